// kernels_eval.cuh -- sm_100a kernels of ffsat_eval (steps A4-A7 of DESIGN.md).
//
//   fast_tiled_kernel   A4-A6 (+ fused A9 count) for the product fast paths (OR/AND/NAE/XOR kinds,
//                       PAPER.md footnote P:964 and App. B) when n fits shared memory: a CTA
//                       owns 32 points (lane = point) x a range of work units; x tile and gradient
//                       tile live in smem; per-literal terms are staged in var-sorted rows and summed
//                       per variable in ascending slot order (deterministic, no float atomics; the
//                       paper's atomicAdd P:318 is replaced).
//   fast_global_kernel  same products for large n: x transposed [n][B], terms to T[slot][B] in HBM.
//   sym_kernel<G>       root-of-unity product path (Alg. 2 / Eqs. 7-9, in the probability
//                       basis of DESIGN.md) with the gradient from exclusive prefix/suffix products
//                       (Prop. 1 / Eq. 10); G threads per (constraint, point) own literal
//                       chunks and scan chunk products across the group (Prop. 2's log-depth schedule).
//   reduce_grad_kernel  A7: grad[b][v] = sum of per-chunk partials + sum over the variable's T slots in
//                       ascending order, fp64 accumulation, transposed write through smem.
//   reduce_f_kernel     A7: f[b] and unsat[b] in a fixed order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ffsat {
namespace dev {

__device__ __forceinline__ float fmaT(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double fmaT(double a, double b, double c) { return ::fma(a, b, c); }
__device__ __forceinline__ float clamp1(float v) { return fminf(fmaxf(v, -1.0f), 1.0f); }
__device__ __forceinline__ double clamp1(double v) { return fmin(fmax(v, -1.0), 1.0); }

template <typename T>
struct cplx {
    T re, im;
};
template <typename T>
__device__ __forceinline__ cplx<T> cmul(const cplx<T>& a, const cplx<T>& b) {
    return {fmaT(a.re, b.re, -a.im * b.im), fmaT(a.re, b.im, a.im * b.re)};
}

struct FastBucketDev {
    int32_t k, kp, nch, pad0;
    int64_t pos_begin, word_off, slot_off;
    double g0;
    double c0[2], c1[2], g[2];   // channel factor a = c0 + c1 * l, FE += g * prod a
    int32_t tmin, tmax, parity, pad1;
};

struct UnitDev {                 // a run of constraints of one bucket (tiled: one staging batch)
    int32_t bucket, seg_begin, seg_end, rows;
    int64_t pos_begin, pos_end;
};

struct SymSigDev {
    int32_t k, Mp, tmin, tmax, parity, pad;
    int64_t coef_off;
    double g0;
};

__device__ __forceinline__ bool rule_sat(int t, int tmin, int tmax, int parity) {
    bool ok = t >= tmin && t <= tmax;
    if (parity == 1) ok = ok && (t & 1);
    if (parity == 2) ok = ok && !(t & 1);
    return ok;
}

// ------------------------------------------------------------------------------------------------
// Per-clause fast products for one lane (= one point).  l_i = s_i x_{v_i}; channel c factor
// a_i = c0 + c1 l_i; FE = g0 + sum_c g_c prod_i a_i; dFE/dl_i = sum_c g_c c1 prod_{j != i} a_j
// by exclusive prefix/suffix products (no division).  K <= 16 fully unrolled in registers.
template <typename T, int K, int NCH>
__device__ __forceinline__ void fast_terms(const T (&l)[K], const FastBucketDev& bk, T (&term)[K], T& fe) {
    fe = (T)bk.g0;
#pragma unroll
    for (int i = 0; i < K; ++i) term[i] = (T)0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const T c0 = (T)bk.c0[c], c1 = (T)bk.c1[c], g = (T)bk.g[c];
        T a[K], pre[K];
        T run = (T)1;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            a[i] = fmaT(c1, l[i], c0);
            pre[i] = run;
            run *= a[i];
        }
        fe = fmaT(g, run, fe);
        T suf = g * c1;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            term[i] = fmaT(pre[i], suf, term[i]);
            suf *= a[i];
        }
    }
}

// 16 < k <= 64: literals in register blocks of 16 with a prefix checkpoint per block.
// getl(i) returns l_i; addterm(i, v, first) stores (first) or accumulates v into literal i's term.
template <typename T, int NCH, typename GetL, typename AddTerm>
__device__ __forceinline__ void fast_terms_blocked(int k, const FastBucketDev& bk, GetL getl, AddTerm addterm, T& fe) {
    fe = (T)bk.g0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const T c0 = (T)bk.c0[c], c1 = (T)bk.c1[c], g = (T)bk.g[c];
        T chk[4];
        T run = (T)1;
#pragma unroll
        for (int blk = 0; blk < 4; ++blk) {
            chk[blk] = run;
            const int hi = min(k, blk * 16 + 16);
            for (int i = blk * 16; i < hi; ++i) run *= fmaT(c1, getl(i), c0);
        }
        fe = fmaT(g, run, fe);
        T suf = g * c1;
#pragma unroll
        for (int blk = 3; blk >= 0; --blk) {
            const int lo = blk * 16;
            if (lo >= k) continue;
            const int hi = min(k, lo + 16);
            T a[16], pre[16];
            T r = chk[blk];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if (lo + j < hi) {
                    a[j] = fmaT(c1, getl(lo + j), c0);
                    pre[j] = r;
                    r *= a[j];
                }
            }
#pragma unroll
            for (int j = 15; j >= 0; --j) {
                if (lo + j < hi) {
                    addterm(lo + j, pre[j] * suf, c == 0);
                    suf *= a[j];
                }
            }
        }
    }
    if (NCH == 0)
        for (int i = 0; i < k; ++i) addterm(i, (T)0, true);
}

// ------------------------------------------------------------------------------------------------
// Tiled fast kernel.  grid = (ceil(B/32), n_chunks); block = NT threads (NT/32 warps).
template <typename T>
struct TiledArgs {
    const T* x;                  // [B][n]
    int64_t B;
    int32_t n, stage_rows;
    const uint32_t* words;       // var | row << 16 | neg << 31, padded rows of kp words
    const UnitDev* units;
    const uint2* segs;           // (var, row_begin | row_end << 16)
    const FastBucketDev* buckets;
    const int32_t* chunk_units;  // [n_chunks + 1]
    const T* w_pos;              // weights by constraint position
    T* P;                        // [n_chunks][n][B] partial gradients
    double* fpart;               // [n_chunks][B]
    int32_t* upart;              // [n_chunks][B]
};

template <typename T, int K, int NCH>
__device__ __forceinline__ void tiled_clause(const TiledArgs<T>& a, const FastBucketDev& bk, int64_t pos,
                                             const T* xs, T* Ts, int lane, double& facc, int& uacc) {
    const uint32_t* wp = a.words + bk.word_off + (pos - bk.pos_begin) * bk.kp;
    uint32_t w[K];
#pragma unroll
    for (int i = 0; i < K; i += 4) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(wp + i));
        w[i] = q.x;
        if (i + 1 < K) w[i + 1] = q.y;
        if (i + 2 < K) w[i + 2] = q.z;
        if (i + 3 < K) w[i + 3] = q.w;
    }
    T l[K];
    int t = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        T xv = xs[(w[i] & 0xffffu) * 33 + lane];
        bool neg = w[i] >> 31;
        l[i] = neg ? -xv : xv;
        t += (int)((xv < (T)0) != neg);
    }
    T term[K], fe;
    fast_terms<T, K, NCH>(l, bk, term, fe);
    const T wc = a.w_pos[pos];
#pragma unroll
    for (int i = 0; i < K; ++i) {
        T v = wc * term[i];
        Ts[((w[i] >> 16) & 0x7fffu) * 32 + lane] = (w[i] >> 31) ? -v : v;
    }
    facc += (double)(wc * fe);
    uacc += rule_sat(t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

template <typename T, int NCH, int KMAX>
__device__ void tiled_clause_dispatch(const TiledArgs<T>& a, const FastBucketDev& bk, int64_t pos, const T* xs, T* Ts,
                                      int lane, double& facc, int& uacc) {
    switch (bk.k) {
#define FFSAT_K(KK) case KK: if (KK <= KMAX) { tiled_clause<T, (KK <= KMAX ? KK : 1), NCH>(a, bk, pos, xs, Ts, lane, facc, uacc); return; } break;
        FFSAT_K(1) FFSAT_K(2) FFSAT_K(3) FFSAT_K(4) FFSAT_K(5) FFSAT_K(6) FFSAT_K(7) FFSAT_K(8)
        FFSAT_K(9) FFSAT_K(10) FFSAT_K(11) FFSAT_K(12) FFSAT_K(13) FFSAT_K(14) FFSAT_K(15) FFSAT_K(16)
#undef FFSAT_K
    default: break;
    }
    if (KMAX <= 16) return;
    // 16 < k <= 64: literal values re-read from the x tile, terms accumulated in their staging rows
    const int k = bk.k;
    const uint32_t* wp = a.words + bk.word_off + (pos - bk.pos_begin) * bk.kp;
    int t = 0;
    for (int i = 0; i < k; ++i) {
        uint32_t w = __ldg(wp + i);
        T xv = xs[(w & 0xffffu) * 33 + lane];
        t += (int)((xv < (T)0) != (bool)(w >> 31));
    }
    auto getl = [&](int i) -> T {
        uint32_t w = __ldg(wp + i);
        T xv = xs[(w & 0xffffu) * 33 + lane];
        return (w >> 31) ? -xv : xv;
    };
    auto addterm = [&](int i, T v, bool first) {
        uint32_t w = __ldg(wp + i);
        T* dst = Ts + ((w >> 16) & 0x7fffu) * 32 + lane;
        *dst = first ? v : *dst + v;
    };
    T fe;
    fast_terms_blocked<T, NCH>(k, bk, getl, addterm, fe);
    const T wc = a.w_pos[pos];
    for (int i = 0; i < k; ++i) {
        uint32_t w = __ldg(wp + i);
        T* dst = Ts + ((w >> 16) & 0x7fffu) * 32 + lane;
        T v = wc * *dst;
        *dst = (w >> 31) ? -v : v;
    }
    facc += (double)(wc * fe);
    uacc += rule_sat(t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(256) fast_tiled_kernel(TiledArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int n = a.n;
    T* xs = reinterpret_cast<T*>(smem_raw);                 // [n][33]
    T* Gs = xs + (size_t)n * 33;                            // [n][33]
    T* Ts = Gs + (size_t)n * 33;                            // [stage_rows][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * 32;
    const int64_t b = b0 + lane;
    const int chunk = blockIdx.y;

    for (int idx = threadIdx.x; idx < 32 * n; idx += blockDim.x) {
        int r = idx / n, v = idx - r * n;
        int64_t bb = b0 + r;
        xs[v * 33 + r] = bb < a.B ? a.x[bb * n + v] : (T)0;
        Gs[v * 33 + r] = (T)0;
    }
    __syncthreads();

    double facc = 0.0;
    int uacc = 0;
    const int u0 = a.chunk_units[chunk], u1 = a.chunk_units[chunk + 1];
    for (int u = u0; u < u1; ++u) {
        const UnitDev U = a.units[u];
        const FastBucketDev bk = a.buckets[U.bucket];
        for (int64_t pos = U.pos_begin + warp; pos < U.pos_end; pos += nw) {
            if (bk.nch == 1) tiled_clause_dispatch<T, 1, KMAX>(a, bk, pos, xs, Ts, lane, facc, uacc);
            else if (bk.nch == 2) tiled_clause_dispatch<T, 2, KMAX>(a, bk, pos, xs, Ts, lane, facc, uacc);
            else tiled_clause_dispatch<T, 0, KMAX>(a, bk, pos, xs, Ts, lane, facc, uacc);
        }
        __syncthreads();
        for (int s = U.seg_begin + warp; s < U.seg_end; s += nw) {
            uint2 sg = __ldg(a.segs + s);
            int rb = sg.y & 0xffffu, re = sg.y >> 16;
            T acc = (T)0;
            for (int r = rb; r < re; ++r) acc += Ts[r * 32 + lane];
            Gs[sg.x * 33 + lane] += acc;
        }
        __syncthreads();
    }
    // outputs: partial gradient tile, partial f / unsat (fixed warp order)
    if (b < a.B) {
        for (int v = warp; v < n; v += nw) a.P[((int64_t)chunk * n + v) * a.B + b] = Gs[v * 33 + lane];
    }
    double* fr = reinterpret_cast<double*>(Ts);   // reuse staging
    int* ur = reinterpret_cast<int*>(fr + nw * 32);
    fr[warp * 32 + lane] = facc;
    ur[warp * 32 + lane] = uacc;
    __syncthreads();
    if (warp == 0 && b < a.B) {
        double f = 0.0;
        int uc = 0;
        for (int w = 0; w < nw; ++w) {
            f += fr[w * 32 + lane];
            uc += ur[w * 32 + lane];
        }
        a.fpart[(int64_t)chunk * a.B + b] = f;
        a.upart[(int64_t)chunk * a.B + b] = uc;
    }
}

// ------------------------------------------------------------------------------------------------
// Global fast kernel (large n).  grid = (ceil(B/32), n_chunks); block = 256.  xT [n][B].
template <typename T>
struct GlobalArgs {
    const T* xT;                 // [n][B]
    int64_t B;
    int32_t n;
    const uint32_t* words;       // var | neg << 31, padded rows
    const UnitDev* units;
    const FastBucketDev* buckets;
    const int32_t* chunk_units;
    const T* w_pos;
    T* Tb;                       // [tb_slots][B]
    double* fpart;
    int32_t* upart;
};

template <typename T, int K, int NCH>
__device__ __forceinline__ void global_clause(const GlobalArgs<T>& a, const FastBucketDev& bk, int64_t pos, int64_t b,
                                              bool bv, double& facc, int& uacc) {
    const uint32_t* wp = a.words + bk.word_off + (pos - bk.pos_begin) * bk.kp;
    uint32_t w[K];
#pragma unroll
    for (int i = 0; i < K; i += 4) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(wp + i));
        w[i] = q.x;
        if (i + 1 < K) w[i + 1] = q.y;
        if (i + 2 < K) w[i + 2] = q.z;
        if (i + 3 < K) w[i + 3] = q.w;
    }
    T l[K];
    int t = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        T xv = bv ? a.xT[(int64_t)(w[i] & 0x7fffffffu) * a.B + b] : (T)0;
        bool neg = w[i] >> 31;
        l[i] = neg ? -xv : xv;
        t += (int)((xv < (T)0) != neg);
    }
    T term[K], fe;
    fast_terms<T, K, NCH>(l, bk, term, fe);
    const T wc = a.w_pos[pos];
    const int64_t slot0 = bk.slot_off + (pos - bk.pos_begin) * bk.k;
    if (bv) {
#pragma unroll
        for (int i = 0; i < K; ++i) {
            T v = wc * term[i];
            a.Tb[(slot0 + i) * a.B + b] = (w[i] >> 31) ? -v : v;
        }
    }
    facc += (double)(wc * fe);
    uacc += rule_sat(t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

template <typename T, int NCH, int KMAX>
__device__ void global_clause_dispatch(const GlobalArgs<T>& a, const FastBucketDev& bk, int64_t pos, int64_t b, bool bv,
                                       double& facc, int& uacc) {
    switch (bk.k) {
#define FFSAT_K(KK) case KK: if (KK <= KMAX) { global_clause<T, (KK <= KMAX ? KK : 1), NCH>(a, bk, pos, b, bv, facc, uacc); return; } break;
        FFSAT_K(1) FFSAT_K(2) FFSAT_K(3) FFSAT_K(4) FFSAT_K(5) FFSAT_K(6) FFSAT_K(7) FFSAT_K(8)
        FFSAT_K(9) FFSAT_K(10) FFSAT_K(11) FFSAT_K(12) FFSAT_K(13) FFSAT_K(14) FFSAT_K(15) FFSAT_K(16)
#undef FFSAT_K
    default: break;
    }
    if (KMAX <= 16) return;
    const int k = bk.k;
    const uint32_t* wp = a.words + bk.word_off + (pos - bk.pos_begin) * bk.kp;
    const int64_t slot0 = bk.slot_off + (pos - bk.pos_begin) * bk.k;
    int t = 0;
    for (int i = 0; i < k; ++i) {
        uint32_t w = __ldg(wp + i);
        T xv = bv ? a.xT[(int64_t)(w & 0x7fffffffu) * a.B + b] : (T)0;
        t += (int)((xv < (T)0) != (bool)(w >> 31));
    }
    auto getl = [&](int i) -> T {
        uint32_t w = __ldg(wp + i);
        T xv = bv ? a.xT[(int64_t)(w & 0x7fffffffu) * a.B + b] : (T)0;
        return (w >> 31) ? -xv : xv;
    };
    T dummy = (T)0;
    auto addterm = [&](int i, T v, bool first) {
        T* dst = bv ? a.Tb + (slot0 + i) * a.B + b : &dummy;
        *dst = first ? v : *dst + v;
    };
    T fe;
    fast_terms_blocked<T, NCH>(k, bk, getl, addterm, fe);
    const T wc = a.w_pos[pos];
    if (bv) {
        for (int i = 0; i < k; ++i) {
            uint32_t w = __ldg(wp + i);
            T* dst = a.Tb + (slot0 + i) * a.B + b;
            T v = wc * *dst;
            *dst = (w >> 31) ? -v : v;
        }
    }
    facc += (double)(wc * fe);
    uacc += rule_sat(t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(256) fast_global_kernel(GlobalArgs<T> a) {
    __shared__ double fr[8 * 32];
    __shared__ int ur[8 * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * 32 + lane;
    const bool bv = b < a.B;
    const int chunk = blockIdx.y;
    double facc = 0.0;
    int uacc = 0;
    for (int u = a.chunk_units[chunk]; u < a.chunk_units[chunk + 1]; ++u) {
        const UnitDev U = a.units[u];
        const FastBucketDev bk = a.buckets[U.bucket];
        for (int64_t pos = U.pos_begin + warp; pos < U.pos_end; pos += nw) {
            if (bk.nch == 1) global_clause_dispatch<T, 1, KMAX>(a, bk, pos, b, bv, facc, uacc);
            else if (bk.nch == 2) global_clause_dispatch<T, 2, KMAX>(a, bk, pos, b, bv, facc, uacc);
            else global_clause_dispatch<T, 0, KMAX>(a, bk, pos, b, bv, facc, uacc);
        }
    }
    fr[warp * 32 + lane] = facc;
    ur[warp * 32 + lane] = uacc;
    __syncthreads();
    if (warp == 0 && bv) {
        double f = 0.0;
        int uc = 0;
        for (int w = 0; w < nw; ++w) {
            f += fr[w * 32 + lane];
            uc += ur[w * 32 + lane];
        }
        a.fpart[(int64_t)chunk * a.B + b] = f;
        a.upart[(int64_t)chunk * a.B + b] = uc;
    }
}

// ------------------------------------------------------------------------------------------------
// Root-of-unity product path for the remaining symmetric constraints.
// Per (constraint c, point b): factors phi_i(m) = alpha_m + beta_m l_i (probability basis: the
// per-root rescaled form of the paper's gamma_i[m] = w^m + x_i, Eq. 7), Q_m = prod_i phi_i(m) (Eq. 8),
// FE = g0 + Re sum_{m=1}^{M'} G_m Q_m (Eq. 9 with the Hermitian half spectrum), and
// dFE/dl_i = Re sum_m H_m pre_i(m) suf_i(m) with H_m = G_m beta_m (Prop. 1).
template <typename T>
struct SymArgs {
    const T* x;                  // points, element (b, v) at x[b * sb + v * sv]
    int64_t sb, sv;
    int64_t B;
    const uint32_t* words;       // var | neg << 31
    const int64_t* off;          // [n_sym + 1]
    const int32_t* sig_of;       // [n_sym]
    const SymSigDev* sigs;
    const T* coef;               // 8 T per root
    const T* w_sym;              // weights of sym constraints (position order, offset by n_fast)
    int64_t tb_fast;             // first sym slot in T
    T* Tb;                       // [tb_slots][B]
    double* fsym;                // [n_sym][B]  w * FE
    int32_t* usym;               // [n_sym][B]  1 if sgn(x) falsifies
};

template <typename T>
__device__ __forceinline__ cplx<T> shfl_up_c(const cplx<T>& v, int d) {
    return {__shfl_up_sync(0xffffffffu, v.re, d), __shfl_up_sync(0xffffffffu, v.im, d)};
}
template <typename T>
__device__ __forceinline__ cplx<T> shfl_down_c(const cplx<T>& v, int d) {
    return {__shfl_down_sync(0xffffffffu, v.re, d), __shfl_down_sync(0xffffffffu, v.im, d)};
}
template <typename T>
__device__ __forceinline__ cplx<T> shfl_c(const cplx<T>& v, int src) {
    return {__shfl_sync(0xffffffffu, v.re, src), __shfl_sync(0xffffffffu, v.im, src)};
}

template <typename T, int G>
__global__ void __launch_bounds__(G == 32 ? 256 : G) sym_kernel(SymArgs<T> a, int64_t s_begin, int64_t s_end) {
    constexpr int CK = 8;
    constexpr int NWG = G / 32;  // warps per group
    __shared__ cplx<T> wt[2][NWG > 1 ? NWG : 1];
    __shared__ int tcnt[NWG > 1 ? NWG : 1];
    const int lane = threadIdx.x & 31;
    int64_t gid;
    int t;
    if (G == 32) {
        gid = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
        t = lane;
    } else {
        gid = blockIdx.x;
        t = threadIdx.x;
    }
    const int64_t ncons = s_end - s_begin;
    if (gid >= ncons * a.B) return;  // G == 32: whole warp exits together; G > 32: whole block
    const int64_t s = s_begin + gid / a.B;
    const int64_t b = gid - (gid / a.B) * a.B;
    const SymSigDev sg = a.sigs[a.sig_of[s]];
    const int k = sg.k;
    const int64_t lo = a.off[s];
    const int ck = (k + G - 1) / G;
    const int i0 = t * ck;

    T l[CK];
    bool neg[CK];
    int tc = 0;
#pragma unroll
    for (int j = 0; j < CK; ++j) {
        int i = i0 + j;
        l[j] = (T)0;
        neg[j] = false;
        if (j < ck && i < k) {
            uint32_t w = __ldg(a.words + lo + i);
            T xv = a.x[b * a.sb + (int64_t)(w & 0x7fffffffu) * a.sv];
            neg[j] = w >> 31;
            l[j] = neg[j] ? -xv : xv;
            tc += (int)((xv < (T)0) != neg[j]);
        }
    }
    T term[CK];
#pragma unroll
    for (int j = 0; j < CK; ++j) term[j] = (T)0;
    double fe_acc = 0.0;
    const T* cf = a.coef + sg.coef_off * 8;
    const cplx<T> one{(T)1, (T)0};
    const int warp = t >> 5;

    for (int m = 0; m < sg.Mp; ++m) {
        const cplx<T> al{__ldg(cf + 8 * m + 0), __ldg(cf + 8 * m + 1)};
        const cplx<T> be{__ldg(cf + 8 * m + 2), __ldg(cf + 8 * m + 3)};
        const cplx<T> Gm{__ldg(cf + 8 * m + 4), __ldg(cf + 8 * m + 5)};
        const cplx<T> Hm{__ldg(cf + 8 * m + 6), __ldg(cf + 8 * m + 7)};
        // backward within the chunk: insuf_j = prod_{j' > j in chunk} phi_j'
        cplx<T> insuf[CK];
        cplx<T> suf = one;
#pragma unroll
        for (int j = CK - 1; j >= 0; --j) {
            insuf[j] = suf;
            if (j < ck && i0 + j < k) {
                cplx<T> ph{fmaT(be.re, l[j], al.re), fmaT(be.im, l[j], al.im)};
                suf = cmul(suf, ph);
            }
        }
        // exclusive prefix / suffix of chunk products across the group (ordered by t)
        cplx<T> ip = suf, is = suf;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            cplx<T> y = shfl_up_c(ip, d);
            if (lane >= d) ip = cmul(y, ip);
            cplx<T> z = shfl_down_c(is, d);
            if (lane + d < 32) is = cmul(is, z);
        }
        cplx<T> P = shfl_up_c(ip, 1), S = shfl_down_c(is, 1);
        if (lane == 0) P = one;
        if (lane == 31) S = one;
        cplx<T> Q = shfl_c(ip, 31);
        if (NWG > 1) {
            if (lane == 31) wt[m & 1][warp] = ip;
            __syncthreads();
            cplx<T> Pw = one, Sw = one, Qa = one;
            for (int w = 0; w < NWG; ++w) {
                cplx<T> v = wt[m & 1][w];
                Qa = cmul(Qa, v);
                if (w < warp) Pw = cmul(Pw, v);
                if (w > warp) Sw = cmul(Sw, v);
            }
            P = cmul(Pw, P);
            S = cmul(S, Sw);
            Q = Qa;
        }
        // forward: pre = H P S prod_{j' < j in chunk} phi_j'; term_j += Re(pre * insuf_j)
        cplx<T> pre = cmul(cmul(Hm, P), S);
#pragma unroll
        for (int j = 0; j < CK; ++j) {
            if (j < ck && i0 + j < k) {
                term[j] = fmaT(pre.re, insuf[j].re, fmaT(-pre.im, insuf[j].im, term[j]));
                cplx<T> ph{fmaT(be.re, l[j], al.re), fmaT(be.im, l[j], al.im)};
                pre = cmul(pre, ph);
            }
        }
        if (t == 0) fe_acc += (double)Gm.re * (double)Q.re - (double)Gm.im * (double)Q.im;
    }
    const T wc = a.w_sym[s];
#pragma unroll
    for (int j = 0; j < CK; ++j) {
        int i = i0 + j;
        if (j < ck && i < k) {
            T v = wc * term[j];
            a.Tb[(a.tb_fast + lo + i) * a.B + b] = neg[j] ? -v : v;
        }
    }
    // true-literal count of sgn(x) over the group
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, d);
    if (NWG > 1) {
        if (lane == 0) tcnt[warp] = tc;
        __syncthreads();
        tc = 0;
        for (int w = 0; w < NWG; ++w) tc += tcnt[w];
    }
    if (t == 0) {
        a.fsym[s * a.B + b] = (double)wc * (sg.g0 + fe_acc);
        a.usym[s * a.B + b] = rule_sat(tc, sg.tmin, sg.tmax, sg.parity) ? 0 : 1;
    }
}

// ------------------------------------------------------------------------------------------------
// A7 reductions.
template <typename T>
struct ReduceArgs {
    int64_t B;
    int32_t n;
    int32_t n_chunks;            // tiled partial tiles (0 on the global path)
    const T* P;                  // [n_chunks][n][B]
    const T* Tb;                 // [tb_slots][B]
    const int64_t* occ_off;      // [n + 1]
    const int32_t* occ_slot;
    T* grad;                     // [B][n]
};

// block (32, 8): tile of 32 variables x 32 points
template <typename T>
__global__ void __launch_bounds__(256) reduce_grad_kernel(ReduceArgs<T> a) {
    __shared__ T tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t b0 = (int64_t)blockIdx.x * 32, v0 = (int64_t)blockIdx.y * 32;
    const int64_t b = b0 + tx;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int vl = ty + 8 * j;
        const int64_t v = v0 + vl;
        double acc = 0.0;
        if (v < a.n && b < a.B) {
            for (int c = 0; c < a.n_chunks; ++c) acc += (double)a.P[((int64_t)c * a.n + v) * a.B + b];
            const int64_t e = a.occ_off[v + 1];
            for (int64_t o = a.occ_off[v]; o < e; ++o) acc += (double)a.Tb[(int64_t)a.occ_slot[o] * a.B + b];
        }
        tile[vl][tx] = (T)acc;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int bl = ty + 8 * j;
        const int64_t bb = b0 + bl, v = v0 + tx;
        if (bb < a.B && v < a.n) a.grad[bb * a.n + v] = tile[tx][bl];
    }
}

struct ReduceFArgs {
    int64_t B;
    int32_t n_parts;             // fast partial rows
    int64_t n_sym;
    const double* fpart;         // [n_parts][B]
    const int32_t* upart;
    const double* fsym;          // [n_sym][B]
    const int32_t* usym;
    double* f;                   // [B]
    int32_t* unsat;              // [B] or null
};

__global__ void reduce_f_kernel(ReduceFArgs a) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= a.B) return;
    double f = 0.0;
    int u = 0;
    for (int c = 0; c < a.n_parts; ++c) {
        f += a.fpart[(int64_t)c * a.B + b];
        u += a.upart[(int64_t)c * a.B + b];
    }
    for (int64_t s = 0; s < a.n_sym; ++s) {
        f += a.fsym[s * a.B + b];
        u += a.usym[s * a.B + b];
    }
    a.f[b] = f;
    if (a.unsat) a.unsat[b] = u;
}

// x [B][n] -> xT [n][B]
template <typename T>
__global__ void __launch_bounds__(256) transpose_kernel(const T* __restrict__ x, T* __restrict__ xT, int64_t B, int32_t n) {
    __shared__ T tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t v0 = (int64_t)blockIdx.x * 32, b0 = (int64_t)blockIdx.y * 32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int64_t b = b0 + ty + 8 * j, v = v0 + tx;
        if (b < B && v < n) tile[ty + 8 * j][tx] = x[b * n + v];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int64_t v = v0 + ty + 8 * j, b = b0 + tx;
        if (b < B && v < n) xT[v * B + b] = tile[tx][ty + 8 * j];
    }
}

}  // namespace dev
}  // namespace ffsat
