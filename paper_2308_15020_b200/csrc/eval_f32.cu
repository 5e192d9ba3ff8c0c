// eval_f32.cu -- ffsat_eval launch code and kernels for the float path.
#include "eval_impl.cuh"

namespace ffsat {
template void eval_device_t<float>(ffsat_ctx*, Scratch&, const float*, int64_t, double*, float*, int32_t*, const float*, cudaStream_t, bool, bool);
template dev::PmReduce<float> pm_reduce_args<float>(const ffsat_ctx*, const Scratch&, int64_t, bool);
template void set_tiled_smem<float>(size_t);
template void set_long_smem<float>();

void set_wide_smem(size_t bytes) {
#define FFSAT_KW(K) for (const void* f : {(const void*)dev::fast_wide_kernel<K, 0, true>, (const void*)dev::fast_wide_kernel<K, 1, true>, \
                                          (const void*)dev::fast_wide_kernel<K, 2, true>, (const void*)dev::fast_wide_kernel<K, 3, true>, \
                                          (const void*)dev::fast_wide_kernel<K, 0, false>}) \
                        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    FFSAT_KW(1) FFSAT_KW(2) FFSAT_KW(3) FFSAT_KW(4) FFSAT_KW(5) FFSAT_KW(6) FFSAT_KW(7) FFSAT_KW(8)
    FFSAT_KW(9) FFSAT_KW(10) FFSAT_KW(11) FFSAT_KW(12) FFSAT_KW(13) FFSAT_KW(14) FFSAT_KW(15) FFSAT_KW(16)
#undef FFSAT_KW
}
void set_tmem_smem(size_t bytes) {
#define FFSAT_KT(K) for (const void* f : {(const void*)dev::fast_tmem_kernel<K, 0, true>, (const void*)dev::fast_tmem_kernel<K, 1, true>, \
                                          (const void*)dev::fast_tmem_kernel<K, 2, true>, (const void*)dev::fast_tmem_kernel<K, 3, true>, \
                                          (const void*)dev::fast_tmem_kernel<K, 0, false>}) \
                        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    FFSAT_KT(1) FFSAT_KT(2) FFSAT_KT(3) FFSAT_KT(4) FFSAT_KT(5) FFSAT_KT(6) FFSAT_KT(7) FFSAT_KT(8)
    FFSAT_KT(9) FFSAT_KT(10) FFSAT_KT(11) FFSAT_KT(12) FFSAT_KT(13) FFSAT_KT(14) FFSAT_KT(15) FFSAT_KT(16)
#undef FFSAT_KT
}
}  // namespace ffsat
