// ctx.hpp -- internal state of libffsat shared by its translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/ffsat.h"
#include "host.hpp"

namespace ffsat {
namespace dev {
template <typename T>
struct SymArgs;
template <typename T>
struct SymSplit;
}

#define CK(call)                                                                                     \
    do {                                                                                             \
        cudaError_t e_ = (call);                                                                     \
        if (e_ != cudaSuccess)                                                                       \
            throw ::ffsat::Error(e_ == cudaErrorMemoryAllocation ? FFSAT_ERR_OOM : FFSAT_ERR_CUDA,   \
                                 std::string(#call) + ": " + cudaGetErrorString(e_));                \
    } while (0)

struct DBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() {
        if (p) cudaFree(p);
    }
    void ensure(size_t b) {
        if (b <= bytes && p) return;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (b == 0) return;
        cudaError_t e = cudaMalloc(&p, b);
        if (e != cudaSuccess) {
            p = nullptr;
            cudaGetLastError();
            throw Error(FFSAT_ERR_OOM, "cudaMalloc(" + std::to_string(b) + "): " + cudaGetErrorString(e));
        }
        bytes = b;
    }
    template <class U>
    U* as() const { return reinterpret_cast<U*>(p); }
};

template <class V>
void upload(DBuf& d, const std::vector<V>& h) {
    d.ensure(std::max<size_t>(h.size() * sizeof(V), 16));
    if (!h.empty()) CK(cudaMemcpy(d.p, h.data(), h.size() * sizeof(V), cudaMemcpyHostToDevice));
}

inline unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Launch with programmatic stream serialization (PDL): the kernel may begin while the previous kernel on `st`
// drains; it must call dev::pdl_wait() before touching that kernel's outputs.  Captured into CUDA graphs as a
// programmatic edge.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

}  // namespace ffsat

#define FFSAT_SIDE_STREAMS 8

namespace ffsat {
// Side streams of one evaluation stream for the concurrent root-path classes and length-class chunk groups (fork /
// join through events, graph-capturable).  Created on first use, outside any capture.
struct Forks {
    cudaStream_t side[FFSAT_SIDE_STREAMS] = {};
    cudaEvent_t ev_fork = nullptr, ev_join[FFSAT_SIDE_STREAMS] = {};
    bool pending_join[FFSAT_SIDE_STREAMS] = {};
    Forks() = default;
    Forks(const Forks&) = delete;
    Forks& operator=(const Forks&) = delete;
    void ensure() {
        if (ev_fork) return;
        for (int i = 0; i < FFSAT_SIDE_STREAMS; ++i) {
            CK(cudaStreamCreateWithFlags(&side[i], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&ev_join[i], cudaEventDisableTiming));
        }
        CK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    }
    ~Forks() {
    }
};
// Per-batch scratch of one evaluation stream: the context's own ffsat_eval calls use ctx->scr (and scr2 for the
// second concurrent host-buffer chunk), every search owns one (so a search's captured CUDA graph never references
// buffers another call may resize); each with its own side streams, so two evaluations can run concurrently.
struct Scratch {
    DBuf xT, Tb, P, fpart, upart, fsym, usym, TbS, fS;
    DBuf tree_ctr;                // work counters of the product-tree classes (one int32 per sym class)
    Forks fk;
    int64_t B = -1;
};
}  // namespace ffsat

struct ffsat_ctx {
    ffsat::Formula F;
    ffsat::Layout Lo;
    int device = -1;
    int num_sm = 148;
    size_t esize = 4;
    std::string err;
    // persistent device layout
    ffsat::DBuf fast_words, tiled_words, units, buckets, sym_words, sym_off, sym_sig, sigs, coef, occ_off, occ_slot,
        w_pos, w_static_orig, order, chk_off, chk_words, chk_rule, chk_long, own_off, own_rec, grp_desc, grp_var, grp_rec;
    int32_t n_chk_long = 0;              // rows longer than dev::kCheckLong (positions in chk_long)
    int64_t persistent_bytes = 0;
    // the batch-independent launch plan (plan_chunks, at load): chunk split of the fast kernels and root splits.
    // It depends on the formula and on batch_ref only -- never on the B of a call -- so every point's f / grad
    // bits are the same whatever batch it is evaluated in (restart sharding over any number of GPUs, F7).
    int64_t batch_ref = 1024;
    ffsat::DBuf chunk_units;
    // root splits: effective S per root-path class and its regions of the split partial buffers
    // (TbS: [S][class literals][B] terms, fS: [S][class constraints][B] Re sum G Q)
    std::vector<int32_t> sym_S;
    std::vector<int64_t> sym_offT, sym_offF;
    int64_t sym_totT = 0, sym_totF = 0;   // per point
    int32_t n_chunks = 0;
    int32_t n_vtiles = 0;                 // owner-computes: 8-variable tiles (their partial f rows, folded to n_fold rows)
    int32_t n_fold = 0;
    int32_t f_groups = 8;                 // interleaved groups of the fixed-order f / unsat reduction (8 or 32)
    // scratch of the context's own evaluations; host-buffer staging
    ffsat::Scratch scr;
    ffsat::Scratch scr2;                  // host-buffer evaluations: the second concurrent chunk's scratch
    cudaStream_t comp2 = nullptr;         // ... and its compute stream
    ffsat::DBuf x_stage, g_stage, f_stage, u_stage, w_stage;
    // global path: chunk groups by bucket length class -- chunks [gchunk[g], gchunk[g + 1]) hold the units with
    // k <= 4 (g = 0), 4 < k <= 16 (g = 1), 16 < k (g = 2, the long kernel); each group is one launch
    int32_t gchunk[4] = {0, 0, 0, 0};
    size_t tiled_smem = 0;
    int64_t launches = 0;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    // host-buffer evaluation: copy streams (H2D, D2H) and per-chunk events of the pipelined staging
    cudaStream_t copy_h2d = nullptr, copy_d2h = nullptr;
    std::vector<cudaEvent_t> ev_h2d, ev_done;
    ffsat::DBuf nf_flag;
    int32_t* nf_host = nullptr;   // pinned
    ~ffsat_ctx() {
        for (cudaEvent_t& e : ev)
            if (e) cudaEventDestroy(e);
        if (copy_h2d) cudaStreamDestroy(copy_h2d);
        if (copy_d2h) cudaStreamDestroy(copy_d2h);
        if (comp2) cudaStreamDestroy(comp2);
        for (cudaEvent_t e : ev_h2d) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_done) cudaEventDestroy(e);
        if (nf_host) cudaFreeHost(nf_host);
    }
};

namespace ffsat {

// The batch-independent launch plan (eval.cu): chunk split of the fast kernels for the reference batch
// c->batch_ref, root splits, kernel shared-memory attributes.  Once, at load.
void plan_chunks(ffsat_ctx* c);
// Size scratch S for batch B (synchronous allocations: never inside a stream capture).
void ensure_scratch(const ffsat_ctx* c, Scratch& S, int64_t B);
// f (fp64), grad (T, may be null), unsat (int32, may be null) at device points x [B][n] under weights w_pos (position
// order); async on st, scratch S (eval_f32.cu / eval_f64.cu).  profiled: record c->ev[0..4] around the phases.
// partials_only: stop before the reductions (the search's fused PGD step reduces the point-major partials itself).
template <typename T>
void eval_device_t(ffsat_ctx* c, Scratch& S, const T* x, int64_t B, double* f, T* grad, int32_t* unsat, const T* w_pos,
                   cudaStream_t st, bool profiled, bool partials_only = false);
namespace dev {
template <typename T>
struct PmReduce;
}
// the reduction arguments of the point-major partials of scratch S (tiled TMEM path)
template <typename T>
dev::PmReduce<T> pm_reduce_args(const ffsat_ctx* c, const Scratch& S, int64_t B, bool unsat);
// allow the tiled kernels of dtype T the dynamic shared memory they need (eval_f32.cu / eval_f64.cu)
template <typename T>
void set_tiled_smem(size_t bytes);
void set_wide_smem(size_t bytes);   // eval_f32.cu
void set_tmem_smem(size_t bytes);   // eval_f32.cu
void launch_tree_class(const SymClass& cl, const dev::SymArgs<double>& a, int max_k, int32_t* counter, int num_sm,
                       cudaStream_t st);   // sym_f64.cu
template <typename T>
void set_long_smem();              // the long global kernel's dynamic shared memory (eval_f32.cu / eval_f64.cu)
// one root-path launch class (sym_f32.cu / sym_f64.cu)
template <typename T>
void launch_sym_class(const SymClass& cl, const dev::SymArgs<T>& a, const dev::SymSplit<T>& sp, cudaStream_t st);

}  // namespace ffsat
