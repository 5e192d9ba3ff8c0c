// sym_f64.cu -- root-of-unity path kernels and launches for the double path.
#include "sym_impl.cuh"

namespace ffsat {
template void launch_sym_class<double>(const SymClass&, const dev::SymArgs<double>&, const dev::SymSplit<double>&, cudaStream_t);
}  // namespace ffsat
