// eval_impl.cuh -- launch orchestration of ffsat_eval (steps A4-A7), instantiated per dtype by
// eval_f32.cu and eval_f64.cu so the two dtypes compile in parallel.
#pragma once
#include <algorithm>

#include "ctx.hpp"
#include "kernels_eval.cuh"

namespace ffsat {

// k shared by every fast bucket when all of them are single-channel products with k <= 16, else 0.
inline int uniform_k(const Layout& L) {
    int k = 0;
    for (const FastBucket& b : L.fbuckets) {
        const int nch = (b.gA != 0) + (b.gB != 0) + (b.gX != 0);
        if (nch != 1 || b.k > 16 || (k != 0 && b.k != k)) return 0;
        k = b.k;
    }
    return k;
}

template <typename T>
void launch_tiled_uniform(int k, dim3 grid, size_t smem, cudaStream_t st, const dev::TiledArgs<T>& a) {
    switch (k) {
#define FFSAT_KU(K) case K: dev::fast_tiled_kernel<T, (K <= 4 ? 4 : K <= 8 ? 8 : 16), K><<<grid, 256, smem, st>>>(a); break;
        FFSAT_KU(1) FFSAT_KU(2) FFSAT_KU(3) FFSAT_KU(4) FFSAT_KU(5) FFSAT_KU(6) FFSAT_KU(7) FFSAT_KU(8)
        FFSAT_KU(9) FFSAT_KU(10) FFSAT_KU(11) FFSAT_KU(12) FFSAT_KU(13) FFSAT_KU(14) FFSAT_KU(15) FFSAT_KU(16)
#undef FFSAT_KU
    default: break;
    }
}

inline void launch_wide(int k, int red, bool check, dim3 grid, size_t smem, cudaStream_t st, const dev::TiledArgs<float>& a) {
    const int sel = check ? red : 4;   // 0-3: truth reduction of the fused check; 4: no check
    switch (k * 8 + sel) {
#define FFSAT_KW(K) case K * 8: dev::fast_wide_kernel<K, 0, true><<<grid, 256, smem, st>>>(a); break; \
                    case K * 8 + 1: dev::fast_wide_kernel<K, 1, true><<<grid, 256, smem, st>>>(a); break; \
                    case K * 8 + 2: dev::fast_wide_kernel<K, 2, true><<<grid, 256, smem, st>>>(a); break; \
                    case K * 8 + 3: dev::fast_wide_kernel<K, 3, true><<<grid, 256, smem, st>>>(a); break; \
                    case K * 8 + 4: dev::fast_wide_kernel<K, 0, false><<<grid, 256, smem, st>>>(a); break;
        FFSAT_KW(1) FFSAT_KW(2) FFSAT_KW(3) FFSAT_KW(4) FFSAT_KW(5) FFSAT_KW(6) FFSAT_KW(7) FFSAT_KW(8)
        FFSAT_KW(9) FFSAT_KW(10) FFSAT_KW(11) FFSAT_KW(12) FFSAT_KW(13) FFSAT_KW(14) FFSAT_KW(15) FFSAT_KW(16)
#undef FFSAT_KW
    default: throw Error(FFSAT_ERR_ARG, "wide tiled kernel needs k <= 16");
    }
}

inline void launch_tmem(int k, int red, bool check, dim3 grid, size_t smem, uint32_t cols, cudaStream_t st,
                        const dev::TiledArgs<float>& a) {
    const int sel = check ? red : 4;
    switch (k * 8 + sel) {
#define FFSAT_KT(K) case K * 8: dev::fast_tmem_kernel<K, 0, true><<<grid, 32 * dev::kTmemWarps, smem, st>>>(a, cols); break; \
                    case K * 8 + 1: dev::fast_tmem_kernel<K, 1, true><<<grid, 32 * dev::kTmemWarps, smem, st>>>(a, cols); break; \
                    case K * 8 + 2: dev::fast_tmem_kernel<K, 2, true><<<grid, 32 * dev::kTmemWarps, smem, st>>>(a, cols); break; \
                    case K * 8 + 3: dev::fast_tmem_kernel<K, 3, true><<<grid, 32 * dev::kTmemWarps, smem, st>>>(a, cols); break; \
                    case K * 8 + 4: dev::fast_tmem_kernel<K, 0, false><<<grid, 32 * dev::kTmemWarps, smem, st>>>(a, cols); break;
        FFSAT_KT(1) FFSAT_KT(2) FFSAT_KT(3) FFSAT_KT(4) FFSAT_KT(5) FFSAT_KT(6) FFSAT_KT(7) FFSAT_KT(8)
        FFSAT_KT(9) FFSAT_KT(10) FFSAT_KT(11) FFSAT_KT(12) FFSAT_KT(13) FFSAT_KT(14) FFSAT_KT(15) FFSAT_KT(16)
#undef FFSAT_KT
    default: throw Error(FFSAT_ERR_ARG, "TMEM tiled kernel needs k <= 16");
    }
}

inline int fast_kmax(const Layout& L) {
    int km = 0;
    for (const FastBucket& b : L.fbuckets) km = std::max(km, b.k);
    return km;
}
// largest k <= 16 among the fast buckets (the short global kernel's register bound)
inline int fast_kmax_short(const Layout& L) {
    int km = 0;
    for (const FastBucket& b : L.fbuckets)
        if (b.k <= 16) km = std::max(km, b.k);
    return km;
}

// f (fp64), grad (T, may be null), unsat (int32, may be null) at device points x [B][n]; async on st.
template <typename T>
dev::PmReduce<T> pm_reduce_args(const ffsat_ctx* c, const Scratch& S, int64_t B, bool unsat) {
    const Layout& L = c->Lo;
    dev::PmReduce<T> r{};
    r.B = B; r.n = L.n; r.n_chunks = L.n_fast > 0 ? c->n_chunks : 0; r.groups = c->f_groups; r.n_sym = L.n_sym;
    r.P = S.P.as<T>(); r.Tb = S.Tb.as<T>(); r.occ_off = c->occ_off.as<int64_t>(); r.occ_slot = c->occ_slot.as<int32_t>();
    r.fpart = S.fpart.as<double>(); r.upart = unsat ? S.upart.as<int32_t>() : nullptr; r.fsym = S.fsym.as<double>();
    r.usym = S.usym.as<int32_t>();
    return r;
}

// Points per thread of owner_grp_kernel for a batch of B points: the layout's choice, except that fp32 batches of at
// most 16 (8) points take 2 (1) per thread (one 16- or 8-point slice instead of a mostly empty 32-point one).  A point's arithmetic
// and summation order do not depend on it (same records, same order): the bits are the same either way.
inline int own_ppt_for(const Layout& L, int64_t B, size_t es) {
    if (es != 4 || L.own_ppt != 4 || L.own_lanes != 8) return L.own_ppt;   // (1 lane: 1 point per thread)
    return B <= 8 ? 1 : B <= 16 ? 2 : 4;
}

// owner_grp_kernel for the bucket's (k, product channels), threads per variable and points per thread (fp32: 4 or 2,
// fp64: 2; 16- or 8-byte gathers)
template <typename T, int K, int NCH, int WPB>
void launch_owner_grp_w(int lanes, int ppt, dim3 grid, cudaStream_t st, const dev::OwnerArgs<T>& o, int32_t bucket) {
    constexpr int P4 = sizeof(T) == 4 ? 4 : 2;
    const dim3 blk(32 * WPB);
    if (lanes == 1) {
        dev::owner_grp_kernel<T, K, NCH, 1, 1, WPB><<<grid, blk, 0, st>>>(o, bucket);
    } else if (ppt == 1 && lanes == 8) {
        dev::owner_grp_kernel<T, K, NCH, 8, 1, WPB><<<grid, blk, 0, st>>>(o, bucket);
    } else if (ppt == 2 || sizeof(T) == 8) {
        if (lanes == 2) dev::owner_grp_kernel<T, K, NCH, 2, 2, WPB><<<grid, blk, 0, st>>>(o, bucket);
        else if (lanes == 4) dev::owner_grp_kernel<T, K, NCH, 4, 2, WPB><<<grid, blk, 0, st>>>(o, bucket);
        else dev::owner_grp_kernel<T, K, NCH, 8, 2, WPB><<<grid, blk, 0, st>>>(o, bucket);
    } else {
        if (lanes == 2) dev::owner_grp_kernel<T, K, NCH, 2, P4, WPB><<<grid, blk, 0, st>>>(o, bucket);
        else if (lanes == 4) dev::owner_grp_kernel<T, K, NCH, 4, P4, WPB><<<grid, blk, 0, st>>>(o, bucket);
        else dev::owner_grp_kernel<T, K, NCH, 8, P4, WPB><<<grid, blk, 0, st>>>(o, bucket);
    }
}
template <typename T, int K, int NCH>
void launch_owner_grp_k(int lanes, int ppt, int wpb, dim3 grid, cudaStream_t st, const dev::OwnerArgs<T>& o, int32_t bucket) {
    if (wpb == 4) launch_owner_grp_w<T, K, NCH, 4>(lanes, ppt, grid, st, o, bucket);
    else if (wpb == 2) launch_owner_grp_w<T, K, NCH, 2>(lanes, ppt, grid, st, o, bucket);
    else if (wpb == 1) launch_owner_grp_w<T, K, NCH, 1>(lanes, ppt, grid, st, o, bucket);
    else launch_owner_grp_w<T, K, NCH, 8>(lanes, ppt, grid, st, o, bucket);
}
template <typename T>
void launch_owner_grp(int key, int lanes, int ppt, int wpb, dim3 grid, cudaStream_t st, const dev::OwnerArgs<T>& o, int32_t bucket) {
    switch (key) {
    case 11: launch_owner_grp_k<T, 1, 1>(lanes, ppt, wpb, grid, st, o, bucket); break;
    case 12: launch_owner_grp_k<T, 1, 2>(lanes, ppt, wpb, grid, st, o, bucket); break;
    case 21: launch_owner_grp_k<T, 2, 1>(lanes, ppt, wpb, grid, st, o, bucket); break;
    case 22: launch_owner_grp_k<T, 2, 2>(lanes, ppt, wpb, grid, st, o, bucket); break;
    case 31: launch_owner_grp_k<T, 3, 1>(lanes, ppt, wpb, grid, st, o, bucket); break;
    default: launch_owner_grp_k<T, 3, 2>(lanes, ppt, wpb, grid, st, o, bucket); break;
    }
}

template <typename T>
void eval_device_t(ffsat_ctx* c, Scratch& S, const T* x, int64_t B, double* f, T* grad, int32_t* unsat, const T* w_pos,
                   cudaStream_t st, bool profiled, bool partials_only) {
    const Layout& L = c->Lo;
    if (B == 0) return;
    ensure_scratch(c, S, B);
    const int64_t PT = (B + 31) / 32;
    auto mark = [&](int i) {
        if (profiled) CK(cudaEventRecord(c->ev[i], st));
    };
    mark(0);
    // x^T [n][B] for the global fast kernel and the thread-per-item root classes (coalesced per-point reads)
    const bool need_xT = L.path == 2 || L.sym_lane;
    if (need_xT && L.n > 0) {
        dim3 tg(blocks_for(L.n, 32), blocks_for(B, 32)), tb(32, 8);
        const int sw = L.own_uni >= 0 ? L.own_lanes * own_ppt_for(L, B, sizeof(T)) : kOwnSlice;   // owner slice width
        if (L.own_sliced && sw == 32) dev::transpose_kernel<T, 32><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        else if (L.own_sliced && sw == 16) dev::transpose_kernel<T, 16><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        else if (L.own_sliced && sw == 8) dev::transpose_kernel<T, 8><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        else if (L.own_sliced && sw == 4) dev::transpose_kernel<T, 4><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        else if (L.own_sliced && sw == 1)   // 1-point slices: x^T is x (a canonicalising copy)
            dev::canon_copy_kernel<T><<<(unsigned)std::min<int64_t>(4 * c->num_sm, blocks_for(B * L.n / (16 / (int64_t)sizeof(T)) + 1, 256)), 256, 0, st>>>(
                x, S.xT.as<T>(), B * (int64_t)L.n);
        else if (L.own_sliced) dev::transpose_kernel<T, kOwnSlice><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        else dev::transpose_kernel<T, 0><<<tg, tb, 0, st>>>(x, S.xT.as<T>(), B, L.n);
        c->launches += 1;
    }
    // root-path classes are independent of the fast kernel (disjoint outputs): off the profiling path they
    // run on forked side streams, concurrently with each other and with the fast kernel
    auto launch_sym_all = [&]() {
        if (L.n_sym == 0) return;
        dev::SymArgs<T> a{};
        a.x = x; a.sb = L.n; a.sv = 1; a.B = B;
        a.words = c->sym_words.as<uint32_t>(); a.off = c->sym_off.as<int64_t>(); a.sig_of = c->sym_sig.as<int32_t>();
        a.sigs = c->sigs.as<dev::SymSigDev>(); a.coef = c->coef.as<T>(); a.w_sym = w_pos + L.n_fast;
        a.tb_fast = L.tb_fast; a.Tb = S.Tb.as<T>(); a.fsym = S.fsym.as<double>(); a.usym = S.usym.as<int32_t>();
        const size_t ncl = L.sym_classes.size();
        const bool fork = ncl > 1 || (!profiled && L.n_fast > 0);
        if (fork) {
            S.fk.ensure();
            CK(cudaEventRecord(S.fk.ev_fork, st));
        }
        dev::SymArgs<T> aT = a;    // thread-per-item classes read x^T
        aT.x = S.xT.as<T>(); aT.sb = 1; aT.sv = B;
        for (size_t i = 0; i < ncl; ++i) {
            cudaStream_t ss = fork ? S.fk.side[i % FFSAT_SIDE_STREAMS] : st;
            if (fork && i < FFSAT_SIDE_STREAMS) CK(cudaStreamWaitEvent(ss, S.fk.ev_fork, 0));
            const SymClass& cl = L.sym_classes[i];
            dev::SymSplit<T> sp{};
            sp.S = c->sym_S[i];
            sp.s_end = cl.end;
            sp.lit0 = cl.lit_begin;
            sp.TbS = S.TbS.as<T>() + c->sym_offT[i] * B;
            sp.fS = S.fS.as<double>() + c->sym_offF[i] * B;
            if (cl.G == kTreeClass) {
                if constexpr (sizeof(T) == 8) {
                    const int max_k = (int)(L.sym_off[(size_t)cl.begin + 1] - L.sym_off[(size_t)cl.begin]);   // sorted longest first
                    launch_tree_class(cl, a, max_k, S.tree_ctr.as<int32_t>() + i, c->num_sm, ss);
                } else {
                    throw Error(FFSAT_ERR_ARG, "product-tree class in an fp32 context");
                }
                c->launches += 1;
                continue;
            }
            launch_sym_class<T>(cl, cl.G == 0 ? aT : a, sp, ss);
            c->launches += sp.S > 1 ? 2 : 1;   // + the split combine
        }
        CK(cudaGetLastError());
        if (fork) {
            for (size_t i = 0; i < std::min<size_t>(ncl, FFSAT_SIDE_STREAMS); ++i) {
                CK(cudaEventRecord(S.fk.ev_join[i], S.fk.side[i]));
                S.fk.pending_join[i] = true;
            }
        }
    };
    auto join_sym = [&]() {
        for (int i = 0; i < FFSAT_SIDE_STREAMS; ++i)
            if (S.fk.pending_join[i]) {
                CK(cudaStreamWaitEvent(st, S.fk.ev_join[i], 0));
                S.fk.pending_join[i] = false;
            }
    };
    if (!profiled) launch_sym_all();
    if (L.n_fast > 0 && c->n_chunks > 0) {
        c->launches += 1;
        if (L.path == 1) {
            dev::TiledArgs<T> a{};
            a.x = x; a.B = B; a.n = L.n;
            a.words = c->tiled_words.as<uint32_t>(); a.units = c->units.as<dev::UnitDev>();
            a.buckets = c->buckets.as<dev::FastBucketDev>(); a.chunk_units = c->chunk_units.as<int32_t>(); a.w_pos = w_pos;
            a.P = S.P.as<T>(); a.fpart = S.fpart.as<double>(); a.upart = S.upart.as<int32_t>();
            dim3 grid((unsigned)PT, (unsigned)c->n_chunks);
            const int km = fast_kmax(L);
            const int ku = uniform_k(L);
            if (L.tmem) {
                if constexpr (sizeof(T) == 4) {
                    dim3 gw((unsigned)((B + 63) / 64), (unsigned)c->n_chunks);
                    dev::TiledArgs<float> at = a;
                    at.words = c->fast_words.as<uint32_t>();   // var | neg << 31 (the TMEM column is 2 var)
                    launch_tmem(ku, L.wide_red, unsat != nullptr, gw, c->tiled_smem, tmem_cols(L.n), st, at);
                }
            } else if (L.wide) {
                if constexpr (sizeof(T) == 4) {
                    dim3 gw((unsigned)((B + 63) / 64), (unsigned)c->n_chunks);
                    launch_wide(ku, L.wide_red, unsat != nullptr, gw, c->tiled_smem, st, a);
                }
            } else if (ku > 0) launch_tiled_uniform<T>(ku, grid, c->tiled_smem, st, a);
            else if (km <= 4) dev::fast_tiled_kernel<T, 4><<<grid, 256, c->tiled_smem, st>>>(a);
            else if (km <= 8) dev::fast_tiled_kernel<T, 8><<<grid, 256, c->tiled_smem, st>>>(a);
            else if (km <= 16) dev::fast_tiled_kernel<T, 16><<<grid, 256, c->tiled_smem, st>>>(a);
            else dev::fast_tiled_kernel<T, 64><<<grid, 256, c->tiled_smem, st>>>(a);
        } else {
            // chunk groups (plan): k <= 4, 4 < k <= 16 (each with its own register bound), k > 16 (long kernel)
            dev::GlobalArgs<T> a{};
            a.xT = S.xT.as<T>(); a.B = B; a.n = L.n; a.words = c->fast_words.as<uint32_t>();
            a.units = c->units.as<dev::UnitDev>(); a.buckets = c->buckets.as<dev::FastBucketDev>();
            a.chunk_units = c->chunk_units.as<int32_t>(); a.w_pos = w_pos; a.Tb = S.Tb.as<T>();
            // the fast terms' T rows fit in L2 (126 MB): plain stores, the reduction reads them back from L2
            a.t_keep = (double)L.tb_fast * (double)B * sizeof(T) <= 100.0 * (1 << 20) ? 1 : 0;
            a.fpart = S.fpart.as<double>(); a.upart = S.upart.as<int32_t>();
            // several groups: off the profiling path groups 1, 2 run on side streams, concurrently with group 0
            // (disjoint chunks, T slots and partial rows); joined with the root-path classes below
            int ngroups = 0;
            for (int g = 0; g < 3; ++g) ngroups += c->gchunk[g + 1] > c->gchunk[g];
            const bool gfork = !profiled && ngroups > 1;
            if (gfork) {
                S.fk.ensure();
                CK(cudaEventRecord(S.fk.ev_fork, st));
            }
            int nl = 0;
            for (int g = 0; g < 3; ++g) {
                const int ng = c->gchunk[g + 1] - c->gchunk[g];
                if (ng == 0) continue;
                if (nl++ > 0) c->launches += 1;
                a.chunk_base = c->gchunk[g];
                dim3 grid((unsigned)PT, (unsigned)ng);
                const int si = FFSAT_SIDE_STREAMS - g;   // side streams 7, 6 (the root classes start at 0)
                cudaStream_t gs = st;
                if (gfork && g > 0) {
                    gs = S.fk.side[si];
                    CK(cudaStreamWaitEvent(gs, S.fk.ev_fork, 0));
                }
                if (g == 0) dev::fast_global_kernel<T, 4><<<grid, 256, 0, gs>>>(a);
                else if (g == 1) {
                    if (fast_kmax_short(L) <= 8) dev::fast_global_kernel<T, 8><<<grid, 256, 0, gs>>>(a);
                    else dev::fast_global_kernel<T, 16><<<grid, 256, 0, gs>>>(a);
                } else {
                    dev::fast_global_long_kernel<T><<<grid, 32 * dev::long_warps<T>(), dev::long_smem_bytes<T>(), gs>>>(a);
                }
                if (gs != st) {
                    CK(cudaEventRecord(S.fk.ev_join[si], gs));
                    S.fk.pending_join[si] = true;
                }
            }
        }
        CK(cudaGetLastError());
    }
    mark(1);
    if (profiled) launch_sym_all();
    join_sym();
    if (partials_only) return;
    mark(2);
    if (L.tmem) {
        // point-major partials of the TMEM kernel: gradient (optional), f and unsat in one reduction kernel, programmatic
        // after the product kernel
        c->launches += 1;
        const dev::PmReduce<T> r = pm_reduce_args<T>(c, S, B, unsat != nullptr);
        const unsigned threads = (unsigned)std::min(256, std::max(32, (L.n + 31) / 32 * 32));
        launch_pdl(dev::reduce_pm_kernel<T>, dim3((unsigned)B), dim3(threads), 0, st, r, grad, f, unsat);
        CK(cudaGetLastError());
        mark(3);
        mark(4);
        return;
    }
    dev::ReduceFArgs rf{};
    rf.B = B; rf.n_parts = L.n_fast > 0 ? c->n_chunks + c->n_fold : 0; rf.n_sym = L.n_sym;
    rf.fpart = S.fpart.as<double>(); rf.upart = S.upart.as<int32_t>(); rf.fsym = S.fsym.as<double>();
    rf.usym = S.usym.as<int32_t>(); rf.f = f; rf.unsat = unsat;
    // tiled path with a gradient: the f / unsat reduction rides in the gradient reduction (variable tile 0), one
    // launch fewer per evaluation; the profiled path keeps them apart so the phases can be timed separately, and
    // the global path keeps them apart (its HBM-bound reduction measured slower with the fused variant, c5)
    const bool fuse = grad && L.n > 0 && !profiled && L.path == 1 && c->f_groups == 8;
    if (L.own && L.n > 0) {
        // global path with owner-computes buckets: one kernel forms their terms per variable and adds the T slots
        // (replaces the gradient reduction); it also writes the short constraints' f / unsat partial rows
        c->launches += 1;
        dev::OwnerArgs<T> o{};
        o.xT = S.xT.as<T>(); o.B = B; o.n = L.n; o.own_off = c->own_off.as<int64_t>(); o.own_rec = c->own_rec.as<uint4>();
        o.row_stride = L.own_sliced ? kOwnSlice : B;
        o.slice_stride = L.own_sliced ? kOwnSlice * (int64_t)L.n : 32;
        o.buckets = c->buckets.as<dev::FastBucketDev>(); o.w_pos = w_pos;
        o.Tb = S.Tb.as<T>(); o.occ_off = c->occ_off.as<int64_t>(); o.occ_slot = c->occ_slot.as<int32_t>(); o.grad = grad;
        o.fpart = S.fpart.as<double>(); o.upart = unsat ? S.upart.as<int32_t>() : nullptr;
        o.row0 = c->n_chunks + c->n_fold;
        if (L.own_sliced && L.own_uni >= 0) {   // one owner bucket: grouped records, coefficients once
            o.grp_desc = c->grp_desc.as<uint4>(); o.grp_var = c->grp_var.as<int32_t>(); o.grp_rec = c->grp_rec.as<uint4>();
            const int ppt = own_ppt_for(L, B, sizeof(T));
            const int sw = L.own_lanes * ppt;
            o.grp_pitch = (uint32_t)(sw * sizeof(T));
            dim3 grid(blocks_for(L.n, 32 * L.own_wpb / L.own_lanes), blocks_for(B, sw));
            const int key = L.fbuckets[(size_t)L.own_uni].k * 10 + fast_nch(L.fbuckets[(size_t)L.own_uni]);
            launch_owner_grp<T>(key, L.own_lanes, ppt, L.own_wpb, grid, st, o, L.own_uni);
        } else if (L.own_sliced) {   // kOwnSlice points x 256 / kOwnSlice variables per block
            dim3 grid(blocks_for(L.n, 256 / kOwnSlice), blocks_for(B, kOwnSlice));
            dev::owner_grad_kernel<T, kOwnSlice><<<grid, 256, 0, st>>>(o);
        } else {
            dim3 grid(blocks_for(L.n, 8), blocks_for(B, 32));
            dev::owner_grad_kernel<T, 32><<<grid, 256, 0, st>>>(o);
        }
        dev::fold_rows_kernel<8><<<dim3((unsigned)c->n_fold, blocks_for(B, 32)), 256, 0, st>>>(
            S.fpart.as<double>(), unsat ? S.upart.as<int32_t>() : nullptr, B, o.row0, c->n_vtiles, c->n_chunks);
        c->launches += 1;
    } else if (grad) {
        c->launches += 1;
        dev::ReduceArgs<T> r{};
        r.B = B; r.n = L.n; r.n_chunks = L.path == 1 ? c->n_chunks : 0; r.P = S.P.as<T>(); r.Tb = S.Tb.as<T>();
        r.occ_off = c->occ_off.as<int64_t>(); r.occ_slot = c->occ_slot.as<int32_t>(); r.grad = grad;
        r.rf = rf;
        dim3 grid(blocks_for(L.n, 8), blocks_for(B, 32)), blk(32, 8);
        // the fused (tiled-path) reduction follows the product kernel programmatically (PDL)
        if (fuse) launch_pdl(dev::reduce_grad_kernel<T, true>, grid, blk, 0, st, r);
        else dev::reduce_grad_kernel<T, false><<<grid, blk, 0, st>>>(r);
    }
    mark(3);
    if (!fuse) {
        c->launches += 1;
        // one warp per interleaved group: the same summation order as the fused variant for every batch size
        if (c->f_groups == 32) dev::reduce_f_kernel<32><<<blocks_for(B, 32), 1024, 0, st>>>(rf);
        else dev::reduce_f_kernel<8><<<blocks_for(B, 32), 256, 0, st>>>(rf);
    }
    CK(cudaGetLastError());
    mark(4);
}


template <typename T>
void set_long_smem() {
    CK(cudaFuncSetAttribute((const void*)dev::fast_global_long_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)dev::long_smem_bytes<T>()));
}

template <typename T>
void set_tiled_smem(size_t bytes) {
    const void* kerns[4 + 16] = {(const void*)dev::fast_tiled_kernel<T, 4>, (const void*)dev::fast_tiled_kernel<T, 8>,
                                 (const void*)dev::fast_tiled_kernel<T, 16>, (const void*)dev::fast_tiled_kernel<T, 64>,
#define FFSAT_KU(K) (const void*)dev::fast_tiled_kernel<T, (K <= 4 ? 4 : K <= 8 ? 8 : 16), K>,
                                 FFSAT_KU(1) FFSAT_KU(2) FFSAT_KU(3) FFSAT_KU(4) FFSAT_KU(5) FFSAT_KU(6) FFSAT_KU(7) FFSAT_KU(8)
                                 FFSAT_KU(9) FFSAT_KU(10) FFSAT_KU(11) FFSAT_KU(12) FFSAT_KU(13) FFSAT_KU(14) FFSAT_KU(15) FFSAT_KU(16)
#undef FFSAT_KU
    };
    for (const void* k : kerns) CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
}

}  // namespace ffsat
