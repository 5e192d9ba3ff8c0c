// eval_f64.cu -- ffsat_eval launch code and kernels for the double path.
#include "eval_impl.cuh"

namespace ffsat {
template void eval_device_t<double>(ffsat_ctx*, Scratch&, const double*, int64_t, double*, double*, int32_t*, const double*, cudaStream_t, bool, bool);
template dev::PmReduce<double> pm_reduce_args<double>(const ffsat_ctx*, const Scratch&, int64_t, bool);
template void set_tiled_smem<double>(size_t);
template void set_long_smem<double>();
}  // namespace ffsat
