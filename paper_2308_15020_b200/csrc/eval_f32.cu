// eval_f32.cu -- ffsat_eval launch code and kernels for the float path.
#include "eval_impl.cuh"

namespace ffsat {
template void eval_device_t<float>(ffsat_ctx*, const float*, int64_t, double*, float*, int32_t*, const float*, cudaStream_t, bool);
template void set_tiled_smem<float>(size_t);
}  // namespace ffsat
