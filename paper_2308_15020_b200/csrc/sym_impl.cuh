// sym_impl.cuh -- launch of the root-of-unity path classes (sym_item_kernel), instantiated per dtype by
// sym_f32.cu / sym_f64.cu (separate translation units: the kernel has one instantiation per (NW, C)).
#pragma once
#include "ctx.hpp"
#include "kernels_eval.cuh"

namespace ffsat {

inline void set_sym_smem(const void* kern, size_t bytes) {
    if (bytes > 40 * 1024) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));  // + static smem must fit 48 KB otherwise
}

// One root-path class launch: a CTA of G threads per (constraint, point) item, C literals per thread.
template <typename T>
void launch_sym_class(const SymClass& cl, const dev::SymArgs<T>& a, const dev::SymSplit<T>& sp, cudaStream_t st) {
    const int64_t items = (cl.end - cl.begin) * a.B;
    if (items == 0) return;
    if (items > INT32_MAX) throw Error(FFSAT_ERR_ARG, "too many root-path items for one launch");
        if (cl.G == 0) {   // thread per item; a.x must be x^T here (sb = 1, sv = B)
        const unsigned nb = (unsigned)((items + 255) / 256);
        switch (cl.C) {
        case 8: dev::sym_lane_kernel<T, 8><<<nb, 256, 0, st>>>(a, cl.begin, items); break;
        case 16: dev::sym_lane_kernel<T, 16><<<nb, 256, 0, st>>>(a, cl.begin, items); break;
        case 32: dev::sym_lane_kernel<T, 32><<<nb, 256, 0, st>>>(a, cl.begin, items); break;
        default: throw Error(FFSAT_ERR_ARG, "unsupported root-path lane class");
        }
        return;
    }
    // root splits: sp.S CTAs per item, each staging its share of the root table
    if ((int64_t)items * sp.S > INT32_MAX) throw Error(FFSAT_ERR_ARG, "too many root-path CTAs for one launch");
    const unsigned gs = (unsigned)(items * sp.S);
    const size_t smem = (size_t)((cl.max_mp + sp.S - 1) / sp.S) * 8 * sizeof(T);   // the largest root share
    switch (cl.G / 32 * 1000 + cl.C * 10 + cl.R) {
#define FFSAT_SYM(NW, C) case NW * 1000 + C * 10 + 1: \
        set_sym_smem((const void*)dev::sym_item_kernel<T, NW, C, 1>, smem); \
        dev::sym_item_kernel<T, NW, C, 1><<<gs, 32 * NW, smem, st>>>(a, sp, cl.begin); break;
        FFSAT_SYM(1, 4) FFSAT_SYM(1, 8) FFSAT_SYM(1, 16) FFSAT_SYM(2, 12) FFSAT_SYM(2, 16)
        FFSAT_SYM(4, 10) FFSAT_SYM(3, 16) FFSAT_SYM(4, 14) FFSAT_SYM(4, 16) FFSAT_SYM(6, 16) FFSAT_SYM(8, 16)
#undef FFSAT_SYM
    default: throw Error(FFSAT_ERR_ARG, "unsupported root-path launch class");
    }
    if (sp.S > 1) {
        const int64_t work = (cl.lit_end - cl.lit_begin + cl.end - cl.begin) * a.B;
        dev::sym_combine_kernel<T><<<(unsigned)std::min<int64_t>(4 * 148, (work + 255) / 256), 256, 0, st>>>(a, sp, cl.begin);
    }
}

}  // namespace ffsat
