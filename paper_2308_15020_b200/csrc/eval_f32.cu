// eval_f32.cu -- ffsat_eval launch code and kernels for the float path.
#include "eval_impl.cuh"

namespace ffsat {
template void eval_device_t<float>(ffsat_ctx*, Scratch&, const float*, int64_t, double*, float*, int32_t*, const float*, cudaStream_t, bool);
template void set_tiled_smem<float>(size_t);
template void set_long_smem<float>();

void set_wide_smem(size_t bytes) {
#define FFSAT_KW(K) for (const void* f : {(const void*)dev::fast_wide_kernel<K, 0>, (const void*)dev::fast_wide_kernel<K, 1>, \
                                          (const void*)dev::fast_wide_kernel<K, 2>, (const void*)dev::fast_wide_kernel<K, 3>}) \
                        CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    FFSAT_KW(1) FFSAT_KW(2) FFSAT_KW(3) FFSAT_KW(4) FFSAT_KW(5) FFSAT_KW(6) FFSAT_KW(7) FFSAT_KW(8)
    FFSAT_KW(9) FFSAT_KW(10) FFSAT_KW(11) FFSAT_KW(12) FFSAT_KW(13) FFSAT_KW(14) FFSAT_KW(15) FFSAT_KW(16)
#undef FFSAT_KW
}
}  // namespace ffsat
