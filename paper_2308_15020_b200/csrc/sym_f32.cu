// sym_f32.cu -- root-of-unity path kernels and launches for the float path.
#include "sym_impl.cuh"

namespace ffsat {
template void launch_sym_class<float>(const SymClass&, const dev::SymArgs<float>&, const dev::SymSplit<float>&, cudaStream_t);
}  // namespace ffsat
