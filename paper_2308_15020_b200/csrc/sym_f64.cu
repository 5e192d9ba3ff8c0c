// sym_f64.cu -- root-of-unity path kernels and launches for the double path.
#include "sym_impl.cuh"
#include "kernels_tree.cuh"

namespace ffsat {
template void launch_sym_class<double>(const SymClass&, const dev::SymArgs<double>&, const dev::SymSplit<double>&, cudaStream_t);

// The product-tree class: persistent CTAs (one per SM, one item at a time, longest constraints first) take the class's
// (constraint, point) items from a counter reset on the stream; dynamic shared memory for the longest constraint.
void launch_tree_class(const SymClass& cl, const dev::SymArgs<double>& a, int max_k, int32_t* counter, int num_sm, cudaStream_t st) {
    const int64_t items = (cl.end - cl.begin) * a.B;
    if (items == 0) return;
    const size_t smem = (size_t)tree::tree_geom(max_k).total * sizeof(double);
    if (smem > tree::kTreeSmemMax) throw Error(FFSAT_ERR_ARG, "product-tree constraint does not fit in shared memory");
    static bool set_on[64] = {};   // the attribute is per device
    int devi = 0;
    CK(cudaGetDevice(&devi));
    if (devi < 0 || devi >= 64 || !set_on[devi]) {
        CK(cudaFuncSetAttribute(dev::sym_tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tree::kTreeSmemMax));
        if (devi >= 0 && devi < 64) set_on[devi] = true;
    }
    CK(cudaMemsetAsync(counter, 0, sizeof(int32_t), st));
    const unsigned grid = (unsigned)std::min<int64_t>(items, num_sm);
    dev::sym_tree_kernel<<<grid, dev::kTreeThreads, smem, st>>>(a, cl.begin, items, counter, (int32_t)(smem / sizeof(double)));
}
}  // namespace ffsat
