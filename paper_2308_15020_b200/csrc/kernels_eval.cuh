// kernels_eval.cuh -- sm_100a kernels of ffsat_eval (steps A4-A7 of DESIGN.md).
//
//   fast_tiled_kernel   A4-A6 (+ fused A9 count) for the product fast paths (OR/AND/NAE/XOR kinds,
//                       PAPER.md footnote P:964 and App. B) when n fits shared memory: a CTA
//                       owns 32 points (lane = point) x a range of var-disjoint constraint classes;
//                       x tile and gradient tile live in smem; warps add literal terms straight into
//                       the gradient tile, one class at a time (deterministic order, no float atomics;
//                       the paper's atomicAdd P:318 is replaced).
//   fast_global_kernel  same products for large n: x transposed [n][B], terms to T[slot][B] in HBM.
//   sym_group_kernel    root-of-unity product path (Alg. 2 / Eqs. 7-9, in the probability
//                       basis of DESIGN.md) with the gradient from exclusive prefix/suffix products
//                       (Prop. 1 / Eq. 10); G threads per (constraint, point) own literal
//                       chunks and scan chunk products across the group (Prop. 2's log-depth schedule).
//   reduce_grad_kernel  A7: grad[b][v] = sum of per-chunk partials + sum over the variable's T slots in
//                       ascending order, fp64 accumulation, transposed write through smem.
//   reduce_f_kernel     A7: f[b] and unsat[b] in a fixed order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels_common.cuh"

namespace ffsat {
namespace dev {

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
template <typename T, int NCH, typename BK, typename GetL, typename AddTerm>
__device__ __forceinline__ void fast_terms_blocked(int k, const BK& bk, GetL getl, AddTerm addterm, T& fe) {
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
// Tiled fast kernel: device helpers (the kernel itself and its design notes follow below).
template <typename T>
struct TiledArgs {
    const T* x;                  // [B][n]
    int64_t B;
    int32_t n;
    const uint32_t* words;       // (var * kTilePitch) | neg << 31, rows of kp words
    const UnitDev* units;
    const FastBucketDev* buckets;
    const int32_t* chunk_units;  // [n_chunks + 1]
    const T* w_pos;              // weights by constraint position
    T* P;                        // [n_chunks][n][B] partial gradients
    double* fpart;               // [n_chunks][B]
    int32_t* upart;              // [n_chunks][B]
};

constexpr int kHalf = 33;        // points per tile half-row + 1 pad
constexpr int kPitch = 2 * kHalf; // == kTilePitch of host.hpp: row v = [x[v][0..32] | G[v][0..32]] (interleaved
                                  // so a literal's gradient slot is its x slot + kHalf: one address, two offsets)

__device__ __forceinline__ float flip_sign(float v, uint32_t w) { return __int_as_float(__float_as_int(v) ^ (int)(w & 0x80000000u)); }
__device__ __forceinline__ double flip_sign(double v, uint32_t w) {
    return __longlong_as_double(__double_as_longlong(v) ^ ((long long)(w & 0x80000000u) << 32));
}
// 1 iff the literal (variable value xv, sign bit of w) is True: (xv < 0) xor negated.  The tiles hold
// canonical zeros (-0.0 stored as +0.0), so the sign bit of xv is exactly "xv < 0" (tie rule: x = 0 is False).
__device__ __forceinline__ uint32_t lit_true(float xv, uint32_t w) { return (__float_as_uint(xv) ^ w) >> 31; }
__device__ __forceinline__ uint32_t lit_true(double xv, uint32_t w) { return ((uint32_t)__double2hiint(xv) ^ w) >> 31; }

// Bucket constants of one work unit, converted to the path dtype once (registers).
template <typename T>
struct BucketReg {
    T g0, c0[2], c1[2], g[2];
    int32_t k, kp, tmin, tmax, parity;
    int64_t pos_begin, word_off, slot_off;
};
template <typename T>
__device__ __forceinline__ BucketReg<T> load_bucket(const FastBucketDev* p) {
    BucketReg<T> r;
    r.g0 = (T)p->g0;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
        r.c0[c] = (T)p->c0[c];
        r.c1[c] = (T)p->c1[c];
        r.g[c] = (T)p->g[c];
    }
    r.k = p->k; r.kp = p->kp; r.tmin = p->tmin; r.tmax = p->tmax; r.parity = p->parity;
    r.pos_begin = p->pos_begin; r.word_off = p->word_off; r.slot_off = p->slot_off;
    return r;
}

// Shared-memory element at byte offset (w << log2 sizeof(T)) from a lane's tile base: the 32-bit shift
// drops the literal's sign bit (bit 31), so one LEA forms the address.
template <typename T>
__device__ __forceinline__ const T* tile_at(const T* base, uint32_t w) {
    return reinterpret_cast<const T*>(reinterpret_cast<const char*>(base) + (uint32_t)(w << (sizeof(T) == 8 ? 3 : 2)));
}
template <typename T>
__device__ __forceinline__ T* tile_at(T* base, uint32_t w) {
    return reinterpret_cast<T*>(reinterpret_cast<char*>(base) + (uint32_t)(w << (sizeof(T) == 8 ? 3 : 2)));
}

// One constraint for one lane (= one point), k <= 16 unrolled, literal words already in registers.
// With c_s = s_i c1 (literal sign folded into the factor slope), a_i = c0 + c_s x_{v_i};
// FE = g0 + sum_ch g prod_i a_i and d f / d x_{v_i} = w sum_ch g c_s prod_{j != i} a_j (exclusive
// prefix * suffix products, no division; Prop. 1 / Eq. 10).  The terms are added straight into
// the shared gradient tile (the unit is var-disjoint, so no other warp touches these rows meanwhile).
template <typename T, int K, int NCH>
__device__ __forceinline__ void tiled_clause(const BucketReg<T>& bk, const uint32_t (&w)[K], T wc, const T* xl, T* gl,
                                             double& facc, int& uacc) {
    T xv[K];
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        xv[i] = *tile_at(xl, w[i]);
        t += lit_true(xv[i], w[i]);
    }
    T fe = bk.g0;
    if (NCH == 1) {
        T cs[K], av[K], pre[K];
        T run = (T)1;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            cs[i] = flip_sign(bk.c1[0], w[i]);
            av[i] = fmaT(cs[i], xv[i], bk.c0[0]);
            pre[i] = run;
            run *= av[i];
        }
        fe = fmaT(bk.g[0], run, fe);
        T suf = bk.g[0] * wc;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            T* g = tile_at(gl, w[i]);
            *g = fmaT(pre[i] * suf, cs[i], *g);
            suf *= av[i];
        }
    } else if (NCH == 2) {
        T gs[K];
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            T cs[K], av[K], pre[K];
            T run = (T)1;
#pragma unroll
            for (int i = 0; i < K; ++i) {
                cs[i] = flip_sign(bk.c1[c], w[i]);
                av[i] = fmaT(cs[i], xv[i], bk.c0[c]);
                pre[i] = run;
                run *= av[i];
            }
            fe = fmaT(bk.g[c], run, fe);
            T suf = bk.g[c] * wc;
#pragma unroll
            for (int i = K - 1; i >= 0; --i) {
                gs[i] = c == 0 ? (pre[i] * suf) * cs[i] : fmaT(pre[i] * suf, cs[i], gs[i]);
                suf *= av[i];
            }
        }
#pragma unroll
        for (int i = 0; i < K; ++i) *tile_at(gl, w[i]) += gs[i];
    }
    facc += (double)(wc * fe);
    uacc += rule_sat((int)t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

#define K_PAD(K) (((K) + 3) / 4 * 4)

// K literal words of one constraint row from global memory (16-byte read-only loads)
template <int K>
__device__ __forceinline__ void load_words(const uint32_t* wp, uint32_t (&w)[K]) {
#pragma unroll
    for (int i = 0; i < K; i += 4) {
        uint4 q = __ldg(reinterpret_cast<const uint4*>(wp + i));
        w[i] = q.x;
        if (i + 1 < K) w[i + 1] = q.y;
        if (i + 2 < K) w[i + 2] = q.z;
        if (i + 3 < K) w[i + 3] = q.w;
    }
}

template <int K>
__device__ __forceinline__ void load_words_smem(const uint32_t* sp, uint32_t (&w)[K]) {
#pragma unroll
    for (int i = 0; i < K; i += 4) {
        uint4 q = *reinterpret_cast<const uint4*>(sp + i);
        w[i] = q.x;
        if (i + 1 < K) w[i + 1] = q.y;
        if (i + 2 < K) w[i + 2] = q.z;
        if (i + 3 < K) w[i + 3] = q.w;
    }
}
// Same, but an opaque (volatile) shared load the compiler cannot merge with an earlier load of the same
// words: used to re-read a row instead of keeping it live in registers across the forward pass.
template <int K>
__device__ __forceinline__ void reload_words_smem(const uint32_t* sp, uint32_t (&w)[K]) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(sp);
#pragma unroll
    for (int i = 0; i < K; i += 4) {
        uint32_t q0, q1, q2, q3;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(q0), "=r"(q1), "=r"(q2), "=r"(q3) : "r"(a + 4 * i));
        w[i] = q0;
        if (i + 1 < K) w[i + 1] = q1;
        if (i + 2 < K) w[i + 2] = q2;
        if (i + 3 < K) w[i + 3] = q3;
    }
}

// Two constraints of one (var-disjoint) unit for one lane, fp32: the pair's factor / prefix / suffix
// chains run side by side in packed f32x2 instructions (FFMA2 / FMUL2, sm_100), which issue two fp32
// lanes of work per instruction slot.  Arithmetic is element-wise identical to tiled_clause (round-to-
// nearest fma / mul per element), so results do not depend on how constraints were paired.
template <int K, int NCH>
__device__ __forceinline__ void tiled_clause_pair(const BucketReg<float>& bk, const uint32_t* sw0, const uint32_t* sw1,
                                                  float wc0, float wc1, const float* xl, float* gl, double& facc, int& uacc) {
    float2 av[K], pre[K];
    float2 fe = make_float2(bk.g0, bk.g0);
    uint32_t t0 = 0, t1 = 0;
    {
        uint32_t w0[K], w1[K];
        load_words_smem<K>(sw0, w0);
        load_words_smem<K>(sw1, w1);
        float2 xv[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
            xv[i].x = *tile_at(xl, w0[i]);
            xv[i].y = *tile_at(xl, w1[i]);
            t0 += lit_true(xv[i].x, w0[i]);
            t1 += lit_true(xv[i].y, w1[i]);
        }
        if (NCH >= 1) {
            const float2 c0 = make_float2(bk.c0[0], bk.c0[0]);
            float2 run = make_float2(1.0f, 1.0f);
#pragma unroll
            for (int i = 0; i < K; ++i) {
                av[i] = __ffma2_rn(make_float2(flip_sign(bk.c1[0], w0[i]), flip_sign(bk.c1[0], w1[i])), xv[i], c0);
                pre[i] = run;
                run = __fmul2_rn(run, av[i]);
            }
            fe = __ffma2_rn(make_float2(bk.g[0], bk.g[0]), run, fe);
        }
        if (NCH == 2) {
            // second channel: products of (c0' + c1' l) kept as the prefix / factor arrays of channel 1;
            // channel 0's terms are folded into the gradient tile below before these are overwritten
            float2 suf = make_float2(bk.g[0] * wc0, bk.g[0] * wc1);
#pragma unroll
            for (int i = K - 1; i >= 0; --i) {
                const float2 cs = make_float2(flip_sign(bk.c1[0], w0[i]), flip_sign(bk.c1[0], w1[i]));
                float* g0p = tile_at(gl, w0[i]);
                float* g1p = tile_at(gl, w1[i]);
                float2 gv = make_float2(*g0p, *g1p);
                gv = __ffma2_rn(__fmul2_rn(pre[i], suf), cs, gv);
                *g0p = gv.x;
                *g1p = gv.y;
                suf = __fmul2_rn(suf, av[i]);
            }
            const float2 c0 = make_float2(bk.c0[1], bk.c0[1]);
            float2 run = make_float2(1.0f, 1.0f);
#pragma unroll
            for (int i = 0; i < K; ++i) {
                av[i] = __ffma2_rn(make_float2(flip_sign(bk.c1[1], w0[i]), flip_sign(bk.c1[1], w1[i])), xv[i], c0);
                pre[i] = run;
                run = __fmul2_rn(run, av[i]);
            }
            fe = __ffma2_rn(make_float2(bk.g[1], bk.g[1]), run, fe);
        }
    }
    if (NCH >= 1) {
        // backward sweep of the last channel: literal words re-read from the stage buffer (broadcast LDS)
        // so they need not stay live across the forward pass
        constexpr int c = NCH - 1 > 0 ? NCH - 1 : 0;
        uint32_t w0[K], w1[K];
        reload_words_smem<K>(sw0, w0);
        reload_words_smem<K>(sw1, w1);
        float2 suf = make_float2(bk.g[c] * wc0, bk.g[c] * wc1);
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            const float2 cs = make_float2(flip_sign(bk.c1[c], w0[i]), flip_sign(bk.c1[c], w1[i]));
            float* g0p = tile_at(gl, w0[i]);
            float* g1p = tile_at(gl, w1[i]);
            float2 gv = make_float2(*g0p, *g1p);
            gv = __ffma2_rn(__fmul2_rn(pre[i], suf), cs, gv);
            *g0p = gv.x;
            *g1p = gv.y;
            suf = __fmul2_rn(suf, av[i]);
        }
    }
    facc += (double)(wc0 * fe.x);
    facc += (double)(wc1 * fe.y);
    uacc += rule_sat((int)t0, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
    uacc += rule_sat((int)t1, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

template <typename T, int K, int NCH>
__device__ __forceinline__ void tiled_pair(const BucketReg<T>& bk, const uint32_t* sw0, const uint32_t* sw1, T wc0, T wc1,
                                           const T* xl, T* gl, double& facc, int& uacc) {
    if constexpr (sizeof(T) == 4) {
        tiled_clause_pair<K, NCH>(bk, sw0, sw1, wc0, wc1, xl, gl, facc, uacc);
    } else {
        uint32_t w0[K], w1[K];
        load_words_smem<K>(sw0, w0);
        tiled_clause<T, K, NCH>(bk, w0, wc0, xl, gl, facc, uacc);
        load_words_smem<K>(sw1, w1);
        tiled_clause<T, K, NCH>(bk, w1, wc1, xl, gl, facc, uacc);
    }
}

// ---- unit staging: while a unit is processed, the next unit's literal words and weights are copied
//      global -> shared with cp.async (LDGSTS) into the other half of a double buffer.
constexpr int kStageWords = 256;   // kClassCap (16) constraints x 16 words (k <= 16)
constexpr int kStageCons = 16;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem));
}
template <int BYTES>
__device__ __forceinline__ void cp_async_small(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem), "n"(BYTES));
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

template <typename T>
struct TileStage {
    uint32_t words[2][kStageWords];
    T w[2][kStageCons];
};

template <typename T>
__device__ __forceinline__ void stage_unit(const TiledArgs<T>& a, const UnitDev& U, TileStage<T>& st, int buf) {
    const int nwords = min(unit_count(U) * unit_kp(U), kStageWords);
    const int t = threadIdx.x;
    if (t * 4 < nwords) cp_async16(&st.words[buf][t * 4], a.words + (int64_t)U.word_begin + t * 4);
    const int c = t - 64;
    if (c >= 0 && c < min(unit_count(U), kStageCons)) cp_async_small<sizeof(T)>(&st.w[buf][c], a.w_pos + (int64_t)U.pos_begin + c);
}

// Pipeline state: unit `u` (header `cur`) is processed from stage buffer `buf`; unit u + 1 (`next`) is
// staged or in flight into buf ^ 1; the header of unit u + 2 (`after`) is a register prefetch issued a
// whole unit before it is needed.
struct UnitPipe {
    UnitDev cur, next, after;
    int u, buf;
};

// Advance past `cur` (all threads, after processing it).
template <typename T>
__device__ __forceinline__ void pipe_advance(const TiledArgs<T>& a, UnitPipe& P, int u1, TileStage<T>& st) {
    cp_async_wait_all();
    __syncthreads();          // next's words are visible; everybody is done with cur's buffer
    P.u += 1;
    P.cur = P.next;
    P.next = P.after;
    P.buf ^= 1;
    if (P.u + 1 < u1) stage_unit<T>(a, P.next, st, P.buf ^ 1);
    cp_async_commit();
    if (P.u + 2 < u1) P.after = a.units[P.u + 2];
}

// A run of consecutive units of one bucket: for each unit the warp takes constraints j = warp,
// warp + nw, ... (two at a time), literal words and weights read from the stage buffer; the pipeline
// barrier ends the unit.
template <typename T, int K, int NCH>
__device__ __forceinline__ void tiled_run(const TiledArgs<T>& a, int bucket, const BucketReg<T>& bk, UnitPipe& P, int u1,
                                          TileStage<T>& st, const T* xl, T* gl, int warp, int nw, double& facc, int& uacc) {
    while (P.u < u1 && P.cur.bucket == bucket) {
        const uint32_t* sw = st.words[P.buf];
        const T* swt = st.w[P.buf];
        const int count = unit_count(P.cur);
        int j = warp;
        for (; j + nw < count; j += 2 * nw)
            tiled_pair<T, K, NCH>(bk, sw + j * K_PAD(K), sw + (j + nw) * K_PAD(K), swt[j], swt[j + nw], xl, gl, facc, uacc);
        if (j < count) {
            uint32_t w0[K];
            load_words_smem<K>(sw + j * K_PAD(K), w0);
            tiled_clause<T, K, NCH>(bk, w0, swt[j], xl, gl, facc, uacc);
        }
        pipe_advance<T>(a, P, u1, st);
    }
}

template <typename T, int NCH>
__device__ void tiled_run_long(const TiledArgs<T>& a, int bucket, const BucketReg<T>& bk, UnitPipe& P, int u1, TileStage<T>& st,
                               const T* xl, T* gl, int warp, int nw, double& facc, int& uacc) {
    const int k = bk.k;
    while (P.u < u1 && P.cur.bucket == bucket) {
        for (int j = warp; j < unit_count(P.cur); j += nw) {
            const int64_t pos = (int64_t)P.cur.pos_begin + j;
            const uint32_t* wp = a.words + (int64_t)P.cur.word_begin + (int64_t)j * unit_kp(P.cur);
            uint32_t t = 0;
            for (int i = 0; i < k; ++i) {
                uint32_t w = __ldg(wp + i);
                t += lit_true(*tile_at(xl, w), w);
            }
            const T wc = a.w_pos[pos];
            auto getl = [&](int i) -> T {
                uint32_t w = __ldg(wp + i);
                return flip_sign(*tile_at(xl, w), w);
            };
            auto addterm = [&](int i, T v, bool) {
                uint32_t w = __ldg(wp + i);
                *tile_at(gl, w) += flip_sign(wc * v, w);
            };
            T fe;
            fast_terms_blocked<T, NCH>(k, bk, getl, addterm, fe);
            facc += (double)(wc * fe);
            uacc += rule_sat((int)t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
        }
        pipe_advance<T>(a, P, u1, st);
    }
}

template <typename T, int NCH, int KMAX>
__device__ __forceinline__ void tiled_run_dispatch(const TiledArgs<T>& a, int bucket, const BucketReg<T>& bk, UnitPipe& P, int u1,
                                                   TileStage<T>& st, const T* xl, T* gl, int warp, int nw, double& facc, int& uacc) {
    switch (bk.k) {
#define FFSAT_K(KK) case KK: if (KK <= KMAX) { tiled_run<T, (KK <= KMAX ? KK : 1), NCH>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc); return; } break;
        FFSAT_K(1) FFSAT_K(2) FFSAT_K(3) FFSAT_K(4) FFSAT_K(5) FFSAT_K(6) FFSAT_K(7) FFSAT_K(8)
        FFSAT_K(9) FFSAT_K(10) FFSAT_K(11) FFSAT_K(12) FFSAT_K(13) FFSAT_K(14) FFSAT_K(15) FFSAT_K(16)
#undef FFSAT_K
    default: break;
    }
    if constexpr (KMAX > 16) {
        tiled_run_long<T, NCH>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc);
    } else {
        while (P.u < u1) pipe_advance<T>(a, P, u1, st);   // unreachable (KMAX >= every k); keeps the barriers matched
    }
}

// Tiled fast kernel (n small enough for the x and gradient tiles to live in shared memory).
// grid = (ceil(B/32), n_chunks); block = 256 threads.  lane = point, warp = constraint.  The work units
// of a chunk are var-disjoint classes (host: disjoint_classes): inside a class no variable occurs twice,
// so the 8 warps add their literal terms straight into the shared gradient tile without races; a
// barrier separates classes.  Every (variable, point) entry is therefore accumulated in one fixed order
// (class order, then literal order) -- deterministic without atomics (the paper's atomicAdd).
// KONLY > 0: every unit has k == KONLY and one product channel (the uniform k-CNF / k-XOR case), so the
// run loop is instantiated for that k alone (no dispatch; registers sized for one k).
template <typename T, int KMAX, int KONLY = 0>
__global__ void __launch_bounds__(256, (sizeof(T) == 4 ? (KMAX <= 8 ? 4 : 2) : (KMAX <= 8 ? 2 : 1))) fast_tiled_kernel(TiledArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];   // >= 3 KB (host: tiled_smem_bytes)
    __shared__ __align__(16) TileStage<T> st;
    const int n = a.n;
    T* xs = reinterpret_cast<T*>(smem_raw);                 // [n][kPitch]: x half-rows
    T* Gs = xs + kHalf;                                     //              gradient half-rows
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * 32;
    const int64_t b = b0 + lane;
    const int chunk = blockIdx.y;

    {   // x tile load, 8 independent global loads in flight per thread
        const int tot = 32 * n;
        for (int base = 0; base < tot; base += 8 * 256) {
            T v8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                const int r = idx / n, v = idx - r * n;
                v8[q] = (idx < tot && b0 + r < a.B) ? __ldg(a.x + (b0 + r) * n + v) : (T)0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                if (idx < tot) {
                    const int r = idx / n, v = idx - r * n;
                    xs[v * kPitch + r] = v8[q] + (T)0;   // + 0 canonicalises -0.0 to +0.0
                    Gs[v * kPitch + r] = (T)0;
                }
            }
        }
    }
    __syncthreads();

    double facc = 0.0;
    int uacc = 0;
    const T* xl = xs + lane;
    T* gl = xs + kHalf + lane;
    const int u0 = a.chunk_units[chunk], u1 = a.chunk_units[chunk + 1];
    UnitPipe P;
    P.u = u0;
    P.buf = 0;
    if (u0 < u1) {
        P.cur = a.units[u0];
        stage_unit<T>(a, P.cur, st, 0);
        if (u0 + 1 < u1) {
            P.next = a.units[u0 + 1];
            stage_unit<T>(a, P.next, st, 1);
        }
        if (u0 + 2 < u1) P.after = a.units[u0 + 2];
    }
    cp_async_commit_wait_all();
    __syncthreads();
    while (P.u < u1) {
        const int bucket = P.cur.bucket;
        const FastBucketDev* bp = a.buckets + bucket;
        const BucketReg<T> bk = load_bucket<T>(bp);
        if constexpr (KONLY > 0) {
            tiled_run<T, KONLY, 1>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc);
            continue;
        }
        const int nch = bp->nch;
        if (nch == 1) tiled_run_dispatch<T, 1, KMAX>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc);
        else if (nch == 2) tiled_run_dispatch<T, 2, KMAX>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc);
        else tiled_run_dispatch<T, 0, KMAX>(a, bucket, bk, P, u1, st, xl, gl, warp, nw, facc, uacc);
    }
    // outputs: partial gradient tile, partial f / unsat (fixed warp order)
    if (b < a.B) {
        for (int v = warp; v < n; v += nw) a.P[((int64_t)chunk * n + v) * a.B + b] = Gs[v * kPitch + lane];
    }
    __syncthreads();
    double* fr = reinterpret_cast<double*>(smem_raw);        // [8][32], reuses the tiles
    int* ur = reinterpret_cast<int*>(fr + 8 * 32);           // [8][32]
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
// Wide tiled kernel (fp32, every fast constraint a single product channel with the same k <= 16, n <= 430):
// as fast_tiled_kernel but each lane owns TWO points (b0 + 2 lane, b0 + 2 lane + 1), so a CTA covers 64
// points.  One literal's address, sign and word serve both points; x and gradient values move as float2
// (LDS.64 / STS.64) and every product runs as one packed f32x2 instruction (FFMA2 / FMUL2) for the two
// points.  Row v of the smem tile = [x of 64 points | 2 pad | gradient of 64 points | 2 pad].
constexpr int kWHalf = 66;
constexpr int kWPitch = 2 * kWHalf;   // == kWidePitch of host.hpp

// RED != 0: every bucket's satisfaction is one bit reduction of the literals' truth bits (sign of x xor the
// literal's sign bit, canonical zeros): one LOP3 per literal and point instead of a count (bk.red: +4 =
// satisfied iff the reduced bit is clear).
template <int RED>
__device__ __forceinline__ uint32_t red_init() { return RED == 2 ? 0xffffffffu : 0u; }
template <int RED>
__device__ __forceinline__ uint32_t red_step(uint32_t m, float xv, uint32_t w) {
    const uint32_t bit = __float_as_uint(xv) ^ w;
    return RED == 1 ? (m | bit) : RED == 2 ? (m & bit) : (m ^ bit);
}

// 32-bit shared-memory float2 access at byte address base + 4 w (the multiply by 4 shifts the literal's
// sign bit out, so one IMAD forms the address)
__device__ __forceinline__ float2 lds2(uint32_t addr) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts2(uint32_t addr, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(v.x), "f"(v.y) : "memory");
}

// NC (1 or 2) clauses of one var-disjoint class for the lane's two points, interleaved: every shared-memory load
// of both clauses is issued before the arithmetic (the clauses share no variable, so the gradient entries of the
// second cannot alias the first's stores) and the two prefix / suffix chains run side by side -- twice the
// instruction-level parallelism of one clause between the class barriers.  CHECK: also the satisfaction bit of
// the rounded points (A9, fused), one LOP3 per literal and point.  fe2 accumulates w * FE of the two points.
template <int K, int RED, bool CHECK, int NC>
__device__ __forceinline__ void wide_clauses(const BucketReg<float>& bk, int redpol, const uint32_t* sw0, const uint32_t* sw1,
                                             float wc0, float wc1, uint32_t xl, float2& fe2, int& u0, int& u1) {
    uint32_t ad[NC][K];
    float cs[NC][K];
    float2 xv[NC][K];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        uint32_t w[K];
        load_words_smem<K>(c == 0 ? sw0 : sw1, w);
#pragma unroll
        for (int i = 0; i < K; ++i) {
            ad[c][i] = xl + (w[i] << 2);
            cs[c][i] = flip_sign(bk.c1[0], w[i]);
        }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) xv[c][i] = lds2(ad[c][i]);
    float2 gv[NC][K];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) gv[c][i] = lds2(ad[c][i] + 4 * kWHalf);
    if (CHECK) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            uint32_t t0 = red_init<RED>(), t1 = red_init<RED>();
#pragma unroll
            for (int i = 0; i < K; ++i) {
                // the literal's sign bit is the sign bit of cs (c1 > 0 is flipped iff negated): cs ^ c1 recovers it
                const uint32_t wneg = __float_as_uint(cs[c][i]) ^ __float_as_uint(bk.c1[0]);
                if (RED == 0) {
                    t0 += lit_true(xv[c][i].x, wneg);
                    t1 += lit_true(xv[c][i].y, wneg);
                } else {
                    t0 = red_step<RED>(t0, xv[c][i].x, wneg);
                    t1 = red_step<RED>(t1, xv[c][i].y, wneg);
                }
            }
            if (RED == 0) {
                u0 += rule_sat((int)t0, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
                u1 += rule_sat((int)t1, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
            } else {   // unsat iff the reduced bit differs from the satisfying value
                u0 += (int)((t0 >> 31) ^ (uint32_t)redpol);
                u1 += (int)((t1 >> 31) ^ (uint32_t)redpol);
            }
        }
    }
    const float2 c0 = make_float2(bk.c0[0], bk.c0[0]);
    float2 av[NC][K], pre[NC][K];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            av[c][i] = __ffma2_rn(make_float2(cs[c][i], cs[c][i]), xv[c][i], c0);
            if (i > 0) pre[c][i] = i == 1 ? av[c][0] : __fmul2_rn(pre[c][i - 1], av[c][i - 1]);   // pre[0] = 1 implicit
        }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const float wc = c == 0 ? wc0 : wc1;
        const float2 run = K == 1 ? av[c][0] : __fmul2_rn(pre[c][K - 1], av[c][K - 1]);
        const float2 fe = __ffma2_rn(make_float2(bk.g[0], bk.g[0]), run, make_float2(bk.g0, bk.g0));
        fe2 = __ffma2_rn(make_float2(wc, wc), fe, fe2);
    }
    float2 suf[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const float sw = bk.g[0] * (c == 0 ? wc0 : wc1);
        suf[c] = make_float2(sw, sw);
    }
#pragma unroll
    for (int i = K - 1; i >= 0; --i)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            gv[c][i] = __ffma2_rn(i == 0 ? suf[c] : __fmul2_rn(pre[c][i], suf[c]), make_float2(cs[c][i], cs[c][i]), gv[c][i]);
            if (i > 0) suf[c] = __fmul2_rn(suf[c], av[c][i]);
        }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) sts2(ad[c][i] + 4 * kWHalf, gv[c][i]);
}

// The staging of a class (literal words + weights) spread over the CTA: lane l < 8 of warp w copies 16-byte word
// chunk 8 w + l (a class holds <= 16 rows of <= 16 words = 64 chunks), lanes 8, 9 copy weights 2 w, 2 w + 1; lane
// 10 of warp 0 copies the header of the class after it into the header ring.
template <int K>
__device__ __forceinline__ void stage_class(const TiledArgs<float>& a, const UnitDev& U, int u, int u1, TileStage<float>& st,
                                            UnitDev* hdr, int buf, int warp, int lane) {
    constexpr int KP = K_PAD(K);
    const int count = unit_count(U);
    const int q = warp * 8 + lane;
    if (lane < 8 && q * 4 < count * KP) cp_async16(&st.words[buf][q * 4], a.words + (int64_t)U.word_begin + q * 4);
    const int j = warp * 2 + (lane - 8);
    if (lane >= 8 && lane < 10 && j < count) cp_async_small<4>(&st.w[buf][j], a.w_pos + (int64_t)U.pos_begin + j);
    if (warp == 0 && lane == 10 && u + 1 < u1) cp_async16(&hdr[(u + 1) & 3], a.units + u + 1);
}

// Wide tiled kernel: 8 warps x 2 points per lane = 64 points per CTA; the chunk's var-disjoint classes (<= 16
// clauses, host kClassCap) one after the other, warp w taking clauses w and w + 8 of a class together, a barrier
// between classes (the gradient tile's fixed accumulation order).  Class headers come through a 4-entry ring in
// shared memory (cp.async two classes ahead), so no register waits on a header load.  CHECK = false: the evaluation
// does not count falsified constraints (PGD iterations between checks), which removes the truth reductions.
template <int K, int RED, bool CHECK>
__global__ void __launch_bounds__(256, 2) fast_wide_kernel(TiledArgs<float> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];   // >= 6 KB (host: wide_smem_bytes)
    __shared__ __align__(16) TileStage<float> st;
    __shared__ __align__(16) UnitDev hdr[4];                     // header ring: class u at hdr[u & 3]
    const int n = a.n;
    float* xs = reinterpret_cast<float*>(smem_raw);              // [n][kWPitch]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * 64;
    const int chunk = blockIdx.y;
    const int u0 = a.chunk_units[chunk], u1 = a.chunk_units[chunk + 1];
    if (u0 < u1) {   // the first two classes' staging overlaps the x tile load
        const UnitDev h0 = a.units[u0];
        if (threadIdx.x == 0) hdr[u0 & 3] = h0;
        stage_class<K>(a, h0, u0, u1, st, hdr, 0, warp, lane);
        if (u0 + 1 < u1) {
            const UnitDev h1 = a.units[u0 + 1];
            stage_class<K>(a, h1, u0 + 1, u1, st, hdr, 1, warp, lane);
        }
    }
    cp_async_commit();

    // x tile load: 8 independent global loads in flight per thread (the loop is latency-bound otherwise)
    {
        const int tot = 64 * n;
        for (int base = 0; base < tot; base += 8 * 256) {
            float v8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                const int r = idx / n, v = idx - r * n;
                v8[q] = (idx < tot && b0 + r < a.B) ? __ldg(a.x + (b0 + r) * n + v) : 0.0f;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                if (idx < tot) {
                    const int r = idx / n, v = idx - r * n;
                    xs[v * kWPitch + r] = v8[q] + 0.0f;   // + 0 canonicalises -0.0
                    xs[v * kWPitch + kWHalf + r] = 0.0f;
                }
            }
        }
    }
    cp_async_wait_all();
    __syncthreads();

    double f0 = 0.0, f1 = 0.0;
    int uc0 = 0, uc1 = 0;
    const uint32_t xl32 = (uint32_t)__cvta_generic_to_shared(xs + 2 * lane);   // this lane's x pair in row 0
    int bucket = -1;
    BucketReg<float> bk{};
    int redpol = 0;   // 1: satisfied iff the reduced bit is set, so unsat = bit ^ 1
    int buf = 0;
    for (int u = u0; u < u1; ++u) {
        const UnitDev cur = hdr[u & 3];
        if (cur.bucket != bucket) {
            bucket = cur.bucket;
            bk = load_bucket<float>(a.buckets + bucket);
            redpol = (a.buckets[bucket].red & 4) ? 0 : 1;
        }
        const uint32_t* sw = st.words[buf];
        const float* swt = st.w[buf];
        const int count = unit_count(cur);
        float2 fe2 = make_float2(0.0f, 0.0f);
        if (warp + 8 < count)
            wide_clauses<K, RED, CHECK, 2>(bk, redpol, sw + warp * K_PAD(K), sw + (warp + 8) * K_PAD(K), swt[warp],
                                           swt[warp + 8], xl32, fe2, uc0, uc1);
        else if (warp < count)
            wide_clauses<K, RED, CHECK, 1>(bk, redpol, sw + warp * K_PAD(K), sw, swt[warp], 0.0f, xl32, fe2, uc0, uc1);
        f0 += (double)fe2.x;
        f1 += (double)fe2.y;
        // advance: class u + 1's words and header u + 2 are in shared memory, everybody is done with this buffer
        cp_async_wait_all();
        __syncthreads();
        buf ^= 1;
        if (u + 2 < u1) stage_class<K>(a, hdr[(u + 2) & 3], u + 2, u1, st, hdr, buf ^ 1, warp, lane);
        cp_async_commit();
    }
    pdl_trigger();   // the gradient reduction may be scheduled now (it waits for this grid to complete)
    // outputs: partial gradient tile (float2 per lane), partial f / unsat (fixed warp order)
    const int64_t b = b0 + 2 * lane;
    for (int v = warp; v < n; v += 8) {
        const float2 g = *reinterpret_cast<const float2*>(xs + v * kWPitch + kWHalf + 2 * lane);
        float* dst = a.P + ((int64_t)chunk * n + v) * a.B + b;
        if (b + 1 < a.B && ((a.B & 1) == 0)) *reinterpret_cast<float2*>(dst) = g;
        else {
            if (b < a.B) dst[0] = g.x;
            if (b + 1 < a.B) dst[1] = g.y;
        }
    }
    __syncthreads();
    double* fr = reinterpret_cast<double*>(smem_raw);         // [8][64], reuses the tiles
    int* ur = reinterpret_cast<int*>(fr + 8 * 64);            // [8][64]
    fr[warp * 64 + 2 * lane] = f0;
    fr[warp * 64 + 2 * lane + 1] = f1;
    ur[warp * 64 + 2 * lane] = uc0;
    ur[warp * 64 + 2 * lane + 1] = uc1;
    __syncthreads();
    if (warp < 2) {
        const int p = warp * 32 + lane;
        const int64_t bp = b0 + p;
        if (bp < a.B) {
            double f = 0.0;
            int uc = 0;
            for (int w = 0; w < 8; ++w) {
                f += fr[w * 64 + p];
                uc += ur[w * 64 + p];
            }
            a.fpart[(int64_t)chunk * a.B + bp] = f;
            if (CHECK) a.upart[(int64_t)chunk * a.B + bp] = uc;
        }
    }
}

// ------------------------------------------------------------------------------------------------
// TMEM tiled kernel (fp32, uniform single-channel k <= 16, n <= 256): the wide kernel's arithmetic with the
// gradient tile in TENSOR MEMORY instead of shared memory.  The gradient read-modify-write of every literal term
// (8 of the 12 bytes per term) leaves the shared-memory pipe, which bound the wide kernel (ncu: L1/TEX ~80 % busy),
// for TMEM's own datapath (tcgen05.ld / tcgen05.st, measured 2.5 SM-cycles per 32-lane x 2-column RMW against 4.0
// for LDS.64 + STS.64, scripts/tmem_probe.cu); shared memory keeps only the x tile reads.
//
// A CTA = 16 warps over 64 points (lane = points 2 l, 2 l + 1, as in the wide kernel).  TMEM lane quadrant q
// (lanes 32 q .. 32 q + 31, reachable only from warps w with w % 4 == q) holds warp group q's private partial gradient
// tile of those 64 points: column 2 v + j = variable v, point 2 l + j of lane l.  Group q (warps q, q + 4, q + 8,
// q + 12) takes classes q, q + 4, q + 8, ... of the chunk; a class's <= 16 clauses go 4 per warp (two interleaved
// pairs) and a named barrier of the group (128 threads) separates its classes -- the fixed accumulation order of
// the tile, deterministic without atomics.  At the end the four quadrant tiles are summed in quadrant order into
// the chunk's partial tile.  One CTA per SM (the allocation is the whole 512-column TMEM when n > 128).
constexpr int kTmemWarps = 16;

__device__ __forceinline__ void tmem_ld2(uint32_t taddr, float2& v) {
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(taddr));
    v = make_float2(__uint_as_float(r0), __uint_as_float(r1));
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, float2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(__float_as_uint(v.x)),
                 "r"(__float_as_uint(v.y)) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void named_bar(int id, int threads) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory"); }

// NC (1 or 2) clauses of a var-disjoint class for the lane's two points; words are var | neg << 31.  x from the
// shared tile (row v at xbase + 256 v), the gradient from / to the quadrant's TMEM columns (tq + 2 v).
template <int K, int RED, bool CHECK, int NC>
__device__ __forceinline__ void tmem_clauses(const BucketReg<float>& bk, int redpol, const uint32_t* sw0, const uint32_t* sw1,
                                             float wc0, float wc1, uint32_t xl, uint32_t tq, float2& fe2, int& u0, int& u1) {
    uint32_t w[NC][K];
#pragma unroll
    for (int c = 0; c < NC; ++c) load_words_smem<K>(c == 0 ? sw0 : sw1, w[c]);
    float2 xv[NC][K], gv[NC][K];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) tmem_ld2(tq + (w[c][i] << 1), gv[c][i]);   // the shift drops the sign bit
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) xv[c][i] = lds2(xl + (w[c][i] << 8));
    float cs[NC][K];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) cs[c][i] = flip_sign(bk.c1[0], w[c][i]);
    if (CHECK) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            uint32_t t0 = red_init<RED>(), t1 = red_init<RED>();
#pragma unroll
            for (int i = 0; i < K; ++i) {
                if (RED == 0) {
                    t0 += lit_true(xv[c][i].x, w[c][i]);
                    t1 += lit_true(xv[c][i].y, w[c][i]);
                } else {
                    t0 = red_step<RED>(t0, xv[c][i].x, w[c][i]);
                    t1 = red_step<RED>(t1, xv[c][i].y, w[c][i]);
                }
            }
            if (RED == 0) {
                u0 += rule_sat((int)t0, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
                u1 += rule_sat((int)t1, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
            } else {
                u0 += (int)((t0 >> 31) ^ (uint32_t)redpol);
                u1 += (int)((t1 >> 31) ^ (uint32_t)redpol);
            }
        }
    }
    const float2 c0 = make_float2(bk.c0[0], bk.c0[0]);
    float2 av[NC][K], pre[NC][K];
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            av[c][i] = __ffma2_rn(make_float2(cs[c][i], cs[c][i]), xv[c][i], c0);
            if (i > 0) pre[c][i] = i == 1 ? av[c][0] : __fmul2_rn(pre[c][i - 1], av[c][i - 1]);
        }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const float wc = c == 0 ? wc0 : wc1;
        const float2 run = K == 1 ? av[c][0] : __fmul2_rn(pre[c][K - 1], av[c][K - 1]);
        const float2 fe = __ffma2_rn(make_float2(bk.g[0], bk.g[0]), run, make_float2(bk.g0, bk.g0));
        fe2 = __ffma2_rn(make_float2(wc, wc), fe, fe2);
    }
    float2 suf[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const float sv = bk.g[0] * (c == 0 ? wc0 : wc1);
        suf[c] = make_float2(sv, sv);
    }
    tmem_wait_ld();
    // the loaded registers are valid only after the wait: pin every use behind it (asm volatile keeps the order)
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) asm volatile("" : "+f"(gv[c][i].x), "+f"(gv[c][i].y));
#pragma unroll
    for (int i = K - 1; i >= 0; --i)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            gv[c][i] = __ffma2_rn(i == 0 ? suf[c] : __fmul2_rn(pre[c][i], suf[c]), make_float2(cs[c][i], cs[c][i]), gv[c][i]);
            if (i > 0) suf[c] = __fmul2_rn(suf[c], av[c][i]);
        }
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
        for (int i = 0; i < K; ++i) tmem_st2(tq + (w[c][i] << 1), gv[c][i]);
}

template <int K, int RED, bool CHECK>
__global__ void __launch_bounds__(32 * kTmemWarps, 1) fast_tmem_kernel(TiledArgs<float> a, uint32_t tcols) {
    // dynamic shared memory: x tile [n][64] fp32, then the chunk's RESIDENT class data -- unit headers, literal words,
    // weights -- staged once (the host sizes the chunks so they fit: plan_chunks); the epilogue tiles reuse it all
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ uint32_t s_tbase;
    const int n = a.n;
    float* xs = reinterpret_cast<float*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int q = warp & 3, r = warp >> 2;   // TMEM lane quadrant / warp group, member of the group
    const int64_t b0 = (int64_t)blockIdx.x * 64;
    const int chunk = blockIdx.y;
    const int u0 = a.chunk_units[chunk], u1 = a.chunk_units[chunk + 1];
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_tbase)), "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    UnitDev* hdr_s = reinterpret_cast<UnitDev*>(smem_raw + (size_t)n * 256);
    uint32_t* words_s = reinterpret_cast<uint32_t*>(hdr_s + (u1 - u0));
    float* w_s = nullptr;
    int wbase = 0, pbase = 0;
    if (u0 < u1) {   // the chunk's units are contiguous in positions and literal words (host layout)
        const UnitDev uf = a.units[u0], ul = a.units[u1 - 1];
        wbase = uf.word_begin;
        pbase = uf.pos_begin;
        const int nwords = ul.word_begin + unit_count(ul) * unit_kp(ul) - wbase;   // a multiple of 4
        const int ncons = ul.pos_begin + unit_count(ul) - pbase;
        w_s = reinterpret_cast<float*>(words_s + nwords);
        for (int i = threadIdx.x; i < u1 - u0; i += blockDim.x) cp_async16(&hdr_s[i], a.units + u0 + i);
        for (int i = threadIdx.x; 4 * i < nwords; i += blockDim.x) cp_async16(&words_s[4 * i], a.words + wbase + 4 * i);
        for (int i = threadIdx.x; i < ncons; i += blockDim.x) cp_async_small<4>(&w_s[i], a.w_pos + pbase + i);
    }
    cp_async_commit();
    {   // x tile [n][64]: row v = 64 points (256 B).  Thread t covers point t % 64, so a warp's 32 stores of one row are
        // 32 consecutive words (bank-conflict-free; the row-major mapping would put a warp's stores 256 B apart, one
        // bank: 32-way conflicts); 16-byte loads of 4 consecutive variables when the rows allow it.
        const int p = (int)threadIdx.x & 63, g0 = (int)threadIdx.x >> 6;   // 8 variable groups per pass
        const bool pv = b0 + p < a.B;
        const float* xr = a.x + (b0 + p) * n;
        if ((n & 3) == 0) {
            for (int v4 = g0; v4 < (n >> 2); v4 += 8) {
                const float4 q4 = pv ? __ldg(reinterpret_cast<const float4*>(xr) + v4) : make_float4(0.f, 0.f, 0.f, 0.f);
                xs[(4 * v4 + 0) * 64 + p] = q4.x + 0.0f;   // + 0 canonicalises -0.0
                xs[(4 * v4 + 1) * 64 + p] = q4.y + 0.0f;
                xs[(4 * v4 + 2) * 64 + p] = q4.z + 0.0f;
                xs[(4 * v4 + 3) * 64 + p] = q4.w + 0.0f;
            }
        } else {
            for (int v = g0; v < n; v += 8) xs[v * 64 + p] = (pv ? __ldg(xr + v) : 0.0f) + 0.0f;
        }
    }
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    const uint32_t tbase = s_tbase;
    const uint32_t tq = tbase + ((uint32_t)(32 * q) << 16);
    // zero the quadrant's 2 n columns (member r takes columns r, r + 4, ... in pairs)
    for (int v = r; v < n; v += 4) tmem_st2(tq + 2 * v, make_float2(0.0f, 0.0f));
    tmem_wait_st();
    cp_async_wait_all();
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();

    double f0 = 0.0, f1 = 0.0;
    int uc0 = 0, uc1 = 0;
    const uint32_t xl32 = (uint32_t)__cvta_generic_to_shared(xs + 2 * lane);
    int bucket = -1;
    BucketReg<float> bk{};
    int redpol = 0;
    // group q takes classes u0 + q, u0 + q + 4, ...; 4 clauses per warp per class as two interleaved pairs; a named
    // barrier per group (128 threads) separates its classes (var-disjoint inside a class: fixed accumulation order)
    for (int u = u0 + q; u < u1; u += 4) {
        const UnitDev cur = hdr_s[u - u0];
        if (cur.bucket != bucket) {
            bucket = cur.bucket;
            bk = load_bucket<float>(a.buckets + bucket);
            redpol = (a.buckets[bucket].red & 4) ? 0 : 1;
        }
        const uint32_t* sw = words_s + (cur.word_begin - wbase);
        const float* swt = w_s + (cur.pos_begin - pbase);
        const int count = unit_count(cur);
        float2 fe2 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {   // clauses r + 8 pr and r + 8 pr + 4
            const int j0 = r + 8 * pr, j1 = j0 + 4;
            if (j1 < count)
                tmem_clauses<K, RED, CHECK, 2>(bk, redpol, sw + j0 * K_PAD(K), sw + j1 * K_PAD(K), swt[j0], swt[j1], xl32, tq,
                                               fe2, uc0, uc1);
            else if (j0 < count)
                tmem_clauses<K, RED, CHECK, 1>(bk, redpol, sw + j0 * K_PAD(K), sw, swt[j0], 0.0f, xl32, tq, fe2, uc0, uc1);
        }
        f0 += (double)fe2.x;
        f1 += (double)fe2.y;
        // end of the class: my TMEM stores are complete before the group's next class
        tmem_wait_st();
        tmem_fence_before();
        named_bar(1 + q, 128);
        tmem_fence_after();
    }
    pdl_trigger();
    // the four quadrant tiles summed in a fixed order, (q0 + q2) + (q1 + q3), through two shared tiles T0 = x tile
    // region, T1 after it (rows of 65 floats: the point-major write-out below reads them conflict-free): round 1
    // q0 -> T0 and q1 -> T1, round 2 q2 += T0 and q3 += T1, then T0 + T1.  Each warp moves 8 variables (16 columns)
    // per tcgen05.ld.
    __syncthreads();
    constexpr int TP = 65;
    float* T0 = xs;              // [n][65]
    float* T1 = xs + n * TP;     // [n][65]
    for (int round = 0; round < 2; ++round) {
        if ((q >> 1) == round) {
            float* T = (q & 1) ? T1 : T0;
            for (int v8 = r * 8; v8 < n; v8 += 32) {   // variables v8 .. v8 + 7 (columns 2 v8 .. 2 v8 + 15)
                uint32_t g[16];
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                             : "=r"(g[0]), "=r"(g[1]), "=r"(g[2]), "=r"(g[3]), "=r"(g[4]), "=r"(g[5]), "=r"(g[6]), "=r"(g[7]),
                               "=r"(g[8]), "=r"(g[9]), "=r"(g[10]), "=r"(g[11]), "=r"(g[12]), "=r"(g[13]), "=r"(g[14]), "=r"(g[15])
                             : "r"(tq + 2 * v8));
                tmem_wait_ld();
#pragma unroll
                for (int j = 0; j < 16; ++j) asm volatile("" : "+r"(g[j]));
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    if (v8 + j < n) {
                        float* dst = T + (v8 + j) * TP + 2 * lane;
                        const float gx = __uint_as_float(g[2 * j]), gy = __uint_as_float(g[2 * j + 1]);
                        if (round == 0) {
                            dst[0] = gx;
                            dst[1] = gy;
                        } else {
                            dst[0] += gx;
                            dst[1] += gy;
                        }
                    }
                }
            }
        }
        tmem_fence_before();
        __syncthreads();
    }
    if (warp == 0) {   // every TMEM access of the CTA is ordered before the deallocation (fence - barrier - fence)
        tmem_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tcols));
    }
    // the chunk's partial gradient, POINT-major: P[chunk][b][v] (a point's row is contiguous, so the reduction -- or
    // the fused PGD step, one CTA per point -- reads it coalesced); warp w writes points w, w + 16, ..., lanes over v
    for (int p = warp; p < 64; p += kTmemWarps) {
        const int64_t bp = b0 + p;
        if (bp >= a.B) break;
        float* dst = a.P + ((int64_t)chunk * a.B + bp) * n;
        for (int v = lane; v < n; v += 32) dst[v] = T0[v * TP + p] + T1[v * TP + p];
    }
    __syncthreads();
    double* fr = reinterpret_cast<double*>(smem_raw);         // [16][64]
    int* ur = reinterpret_cast<int*>(fr + kTmemWarps * 64);   // [16][64]
    fr[warp * 64 + 2 * lane] = f0;
    fr[warp * 64 + 2 * lane + 1] = f1;
    ur[warp * 64 + 2 * lane] = uc0;
    ur[warp * 64 + 2 * lane + 1] = uc1;
    __syncthreads();
    if (warp < 2) {
        const int p = warp * 32 + lane;
        const int64_t bp = b0 + p;
        if (bp < a.B) {
            double f = 0.0;
            int uc = 0;
            for (int w = 0; w < kTmemWarps; ++w) {
                f += fr[w * 64 + p];
                uc += ur[w * 64 + p];
            }
            a.fpart[(int64_t)chunk * a.B + bp] = f;
            if (CHECK) a.upart[(int64_t)chunk * a.B + bp] = uc;
        }
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
    const int32_t* chunk_units;  // [n_chunks + 1]; this launch covers chunks chunk_base + blockIdx.y
    int32_t chunk_base;
    const T* w_pos;
    T* Tb;                       // [tb_slots][B]
    double* fpart;
    int32_t* upart;
    int32_t t_keep;              // 1: the term buffer fits in L2 -- plain stores (the reduction reads it back from L2);
                                 // 0: streaming stores (keep x^T in L2 instead)
};

// T-buffer store: streaming (evict-first) unless the whole buffer fits in L2 and is read back right away
template <typename T>
__device__ __forceinline__ void t_store(T* p, T v, int keep) {
    if (keep) *p = v;
    else __stcs(p, v);
}

// Terms of one constraint for one lane from its literal words and gathered variable values (k <= 16):
// term_i = w d FE / d x_{v_i} (literal sign folded into the factor slope, as in tiled_clause).
template <typename T, int K, int NCH>
__device__ __forceinline__ void clause_terms(const BucketReg<T>& bk, const uint32_t (&w)[K], const T (&xv)[K], T wc, T (&gs)[K],
                                             double& facc, int& uacc) {
    uint32_t t = 0;
#pragma unroll
    for (int i = 0; i < K; ++i) {
        t += (uint32_t)((xv[i] < (T)0) != ((int)w[i] < 0));
        gs[i] = (T)0;
    }
    T fe = bk.g0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        T av[K], pre[K];
        T run = (T)1;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            av[i] = fmaT(flip_sign(bk.c1[c], w[i]), xv[i], bk.c0[c]);
            pre[i] = run;
            run *= av[i];
        }
        fe = fmaT(bk.g[c], run, fe);
        T suf = bk.g[c] * wc;
#pragma unroll
        for (int i = K - 1; i >= 0; --i) {
            gs[i] = fmaT(pre[i] * suf, flip_sign(bk.c1[c], w[i]), gs[i]);
            suf *= av[i];
        }
    }
    facc += (double)(wc * fe);
    uacc += rule_sat((int)t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
}

// One unit on the global path: the warp's constraints two at a time, every load of the pair (literal words,
// then the gathered x^T rows, read-only path) issued before any arithmetic -- the kernel is bound by the
// latency of these gathers and the T stores, so memory-level parallelism is what matters.
template <typename T, int K, int NCH>
__device__ __forceinline__ void global_unit(const GlobalArgs<T>& a, const BucketReg<T>& bk, const UnitDev& U, int64_t b, bool bv,
                                            int warp, int nw, double& facc, int& uacc) {
    // NP constraints of the warp in flight at once (j, j + nw): 2 (4 measured slower on c5: fewer resident warps)
    constexpr int NP = 2;
    const int count = unit_count(U);
    const int64_t wbase = (int64_t)U.word_begin;
    const int64_t sbase = bk.slot_off + ((int64_t)U.pos_begin - bk.pos_begin) * K;
    const int64_t bb = bv ? b : 0;
    for (int j = warp; j < count; j += NP * nw) {
        uint32_t w[NP][K];
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            const int jq = j + q * nw < count ? j + q * nw : j;   // past the unit end: repeat j (not stored)
            load_words<K>(a.words + wbase + (int64_t)jq * K_PAD(K), w[q]);
        }
        T x[NP][K];
#pragma unroll
        for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int i = 0; i < K; ++i) x[q][i] = __ldg(a.xT + (int64_t)(w[q][i] & 0x7fffffffu) * a.B + bb);
        T wc[NP];
#pragma unroll
        for (int q = 0; q < NP; ++q) wc[q] = j + q * nw < count ? __ldg(a.w_pos + U.pos_begin + j + q * nw) : (T)0;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
            if (j + q * nw >= count) break;
            T g[K];
            clause_terms<T, K, NCH>(bk, w[q], x[q], wc[q], g, facc, uacc);
            if (bv) {
#pragma unroll
                for (int i = 0; i < K; ++i) t_store(a.Tb + (sbase + (int64_t)(j + q * nw) * K + i) * a.B + b, g[i], a.t_keep);
            }
        }
    }
}

template <typename T, int NCH, int KMAX>
__device__ __forceinline__ void global_unit_dispatch(const GlobalArgs<T>& a, const BucketReg<T>& bk, const UnitDev& U, int64_t b,
                                                     bool bv, int warp, int nw, double& facc, int& uacc) {
    switch (bk.k) {
#define FFSAT_K(KK) case KK: if (KK <= KMAX) { global_unit<T, (KK <= KMAX ? KK : 1), NCH>(a, bk, U, b, bv, warp, nw, facc, uacc); return; } break;
        FFSAT_K(1) FFSAT_K(2) FFSAT_K(3) FFSAT_K(4) FFSAT_K(5) FFSAT_K(6) FFSAT_K(7) FFSAT_K(8)
        FFSAT_K(9) FFSAT_K(10) FFSAT_K(11) FFSAT_K(12) FFSAT_K(13) FFSAT_K(14) FFSAT_K(15) FFSAT_K(16)
#undef FFSAT_K
    default: break;   // k > 16: fast_global_long_kernel (own chunks)
    }
}

template <typename T, int KMAX>
__global__ void __launch_bounds__(256) fast_global_kernel(GlobalArgs<T> a) {
    __shared__ double fr[8 * 32];
    __shared__ int ur[8 * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * 32 + lane;
    const bool bv = b < a.B;
    const int chunk = a.chunk_base + blockIdx.y;
    double facc = 0.0;
    int uacc = 0;
    int cur = -1;
    BucketReg<T> bk{};
    int nch = 0;
    int base = 0;
    const int ua = a.chunk_units[chunk], ub = a.chunk_units[chunk + 1];
    UnitDev nextU = ua < ub ? a.units[ua] : UnitDev{};
    for (int u = ua; u < ub; ++u) {
        const UnitDev U = nextU;
        if (u + 1 < ub) nextU = a.units[u + 1];   // header of the next unit in flight during this one
        if (U.bucket != cur) {
            cur = U.bucket;
            bk = load_bucket<T>(a.buckets + cur);
            nch = a.buckets[cur].nch;
        }
        // the chunk's constraints are dealt to the warps round-robin across unit boundaries (j0 = this warp's
        // first constraint of the unit), so small units do not idle warps
        const int j0 = ((warp - base) % nw + nw) % nw;
        base += unit_count(U);
        if (nch == 1) global_unit_dispatch<T, 1, KMAX>(a, bk, U, b, bv, j0, nw, facc, uacc);
        else if (nch == 2) global_unit_dispatch<T, 2, KMAX>(a, bk, U, b, bv, j0, nw, facc, uacc);
        else global_unit_dispatch<T, 0, KMAX>(a, bk, U, b, bv, j0, nw, facc, uacc);
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

// Long fast constraints (16 < k <= 64) on the global path: their own launch over the chunks that hold the long
// units (the units are a suffix of the unit list: buckets ascend in k).  Warp = 32 points of one constraint.
// The warp reads the row's literal words once, coalesced (word i in lane i % 32 of register i / 32), and every
// lane issues all k gathers x^T[v_i][b] as 4/8-byte cp.async copies into its own shared column xs[i][lane]
// (no registers held by loads in flight, all k lines requested at once); the exclusive prefixes go to a second
// column; the backward sweep writes every term once (streaming store).  2 warps per CTA (smaller CTAs pack 14 warps per SM), 2 x 64 x 32
// values of shared memory per warp (dynamic: f32 32 KB, f64 64 KB per CTA).
template <typename T>
__host__ __device__ constexpr int long_warps() { return sizeof(T) == 4 ? 2 : 2; }
constexpr int kLongKMax = 64;
template <typename T>
__host__ __device__ constexpr size_t long_smem_bytes() { return (size_t)long_warps<T>() * 2 * kLongKMax * 32 * sizeof(T); }

template <typename T, int NCH>
__device__ void global_unit_long_cp(const GlobalArgs<T>& a, const BucketReg<T>& bk, const UnitDev& U, int64_t b, bool bv,
                                    int j0, T* xs, T* ps, uint32_t* ws, double& facc, int& uacc) {
    const int k = bk.k;
    const int lane = threadIdx.x & 31;
    // lanes past the batch end mirror the last point (same inputs, same arithmetic, same stored values), so the
    // term stores need no predicate: a duplicate lane writes what the last valid lane writes
    const int64_t bb = bv ? b : a.B - 1;
    const char* xb = reinterpret_cast<const char*>(a.xT + bb);
    const size_t rowb = (size_t)a.B * sizeof(T);   // bytes per x^T row (64-bit offsets: any n B)
    for (int j = j0; j < unit_count(U); j += long_warps<T>()) {
        const int64_t pos = (int64_t)U.pos_begin + j;
        const uint32_t* wp = a.words + (int64_t)U.word_begin + (int64_t)j * unit_kp(U);
        const T wc = __ldg(a.w_pos + pos);
        __syncwarp();   // the previous constraint's reads of ws / xs / ps are done
        if (lane < k) ws[lane] = __ldg(wp + lane);
        if (lane + 32 < k) ws[lane + 32] = __ldg(wp + lane + 32);
        __syncwarp();
        // every gather in flight at once: 4/8-byte cp.async per literal into this lane's column (broadcast
        // word reads, one wide multiply-add per address)
#pragma unroll 4
        for (int i = 0; i < k; ++i)
            cp_async_small<sizeof(T)>(xs + 32 * i, xb + (size_t)(ws[i] & 0x7fffffffu) * rowb);
        cp_async_commit_wait_all();
        T fe = bk.g0;
        uint32_t t = 0;
        T* dst = a.Tb + (bk.slot_off + (pos - bk.pos_begin) * k) * a.B + bb;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const T c0 = bk.c0[c], c1 = bk.c1[c];
            T run = (T)1;
            // forward: exclusive prefixes to ps; channel 0 also counts the True literals (x^T holds canonical
            // zeros, so the sign bit of x is exactly x < 0: tie rule x = 0 -> False)
#pragma unroll 4
            for (int i = 0; i < k; ++i) {
                const uint32_t w = ws[i];
                const T xv = xs[32 * i];
                if (c == 0) t += lit_true(xv, w);
                ps[32 * i] = run;
                run *= fmaT(flip_sign(c1, w), xv, c0);
            }
            fe = fmaT(bk.g[c], run, fe);
            T suf = bk.g[c] * wc;
            // backward: term_i = pre_i suf_i s_i c1, written once (channel 0) or accumulated
#pragma unroll 4
            for (int i = k - 1; i >= 0; --i) {
                const uint32_t w = ws[i];
                const T cs = flip_sign(c1, w);
                const T p = ps[32 * i] * suf;
                T* d = dst + (size_t)i * (size_t)a.B;
                if (c == 0) t_store(d, p * cs, a.t_keep);
                else *d = fmaT(p, cs, *d);
                suf *= fmaT(cs, xs[32 * i], c0);
            }
        }
        if (NCH == 0) {
            for (int i = 0; i < k; ++i) {
                t += lit_true(xs[32 * i], ws[i]);
                t_store(dst + (size_t)i * (size_t)a.B, (T)0, a.t_keep);
            }
        }
        facc += (double)(wc * fe);
        uacc += rule_sat((int)t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
    }
}

template <typename T>
__global__ void __launch_bounds__(32 * long_warps<T>()) fast_global_long_kernel(GlobalArgs<T> a) {
    constexpr int kLongWarps = long_warps<T>();
    extern __shared__ __align__(16) unsigned char smem_raw[];   // long_smem_bytes<T>()
    __shared__ double fr[kLongWarps * 32];
    __shared__ int ur[kLongWarps * 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * 32 + lane;
    const bool bv = b < a.B;
    const int chunk = a.chunk_base + blockIdx.y;
    T* xs = reinterpret_cast<T*>(smem_raw) + warp * 2 * kLongKMax * 32 + lane;   // per-lane columns, stride 32
    T* ps = xs + kLongKMax * 32;
    __shared__ uint32_t wsh[kLongWarps][kLongKMax];                                // the warp's row of words
    uint32_t* ws = wsh[warp];
    double facc = 0.0;
    int uacc = 0;
    int cur = -1;
    BucketReg<T> bk{};
    int nch = 0;
    int base = 0;
    const int ua = a.chunk_units[chunk], ub = a.chunk_units[chunk + 1];
    UnitDev nextU = ua < ub ? a.units[ua] : UnitDev{};
    for (int u = ua; u < ub; ++u) {
        const UnitDev U = nextU;
        if (u + 1 < ub) nextU = a.units[u + 1];   // header of the next unit in flight during this one
        if (U.bucket != cur) {
            cur = U.bucket;
            bk = load_bucket<T>(a.buckets + cur);
            nch = a.buckets[cur].nch;
        }
        const int j0 = ((warp - base) % kLongWarps + kLongWarps) % kLongWarps;   // round-robin across units
        base += unit_count(U);
        if (nch == 1) global_unit_long_cp<T, 1>(a, bk, U, b, bv, j0, xs, ps, ws, facc, uacc);
        else if (nch == 2) global_unit_long_cp<T, 2>(a, bk, U, b, bv, j0, xs, ps, ws, facc, uacc);
        else global_unit_long_cp<T, 0>(a, bk, U, b, bv, j0, xs, ps, ws, facc, uacc);
    }
    fr[warp * 32 + lane] = facc;
    ur[warp * 32 + lane] = uacc;
    __syncthreads();
    if (warp == 0 && bv) {
        double f = 0.0;
        int uc = 0;
        for (int w = 0; w < kLongWarps; ++w) {
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

// Root splits (sym_item_kernel, S > 1): CTA (item, split) covers an even share of the item's roots and writes
// partials, summed in split order by sym_combine_kernel.  (A separate kernel argument: growing SymArgs changed
// the code generated for sym_lane_kernel and slowed it by 40%.)
template <typename T>
struct SymSplit {
    int32_t S;
    int64_t s_end, lit0;         // the class's constraint end and first literal
    T* TbS;                      // [S][class literals][B]  w s_i (partial dFE/dl_i)
    double* fS;                  // [S][class constraints][B]  partial Re sum_m G_m Q_m
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

// Root path: one CTA of NW warps per (constraint c, point b) item; thread t owns the C consecutive
// literals [t C, t C + C).  The item index comes from blockIdx alone, so the root loop is uniform and the
// warp shuffles stay convergent.  Launch classes (NW, C) run on forked streams, concurrently with each
// other and with the fast-path kernel, so short and long constraints share waves.  Per root m of the
// Hermitian half spectrum (m = 1..M'):
//   1. backward sweep in registers: factors phi_j = alpha_m + beta_m l_j (probability basis, #2)
//      and exclusive in-chunk suffix products insuf_j; the chunk product;
//   2. exclusive prefix P and suffix S of the chunk products across the group: warp Kogge-Stone scans
//      with shuffles (Prop. 2's log-depth tree), then a named barrier of the group to
//      combine warp totals (NW > 1);
//   3. forward sweep: term_j += Re(A insuf_j) with A = H_m P S prod_{j' < j in chunk} phi_j'.
// FE = g0 + Re sum_m G_m Q_m.  Each literal's term is owned by one thread: no cross-thread gradient sum.
__device__ __forceinline__ void opaque(double& v) { asm volatile("" : "+d"(v)); }
__device__ __forceinline__ void opaque(float& v) { asm volatile("" : "+f"(v)); }

// alpha_m, beta_m of roots m .. m + R - 1 (the last root repeated past Mp; harmless prefetch)
template <typename T, int R>
__device__ __forceinline__ void load_ab(const T* cf, int m, int Mp, cplx<T> (&al)[R], cplx<T> (&be)[R]) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int mm = m + r < Mp ? m + r : Mp - 1;
        al[r] = {cf[8 * mm + 0], cf[8 * mm + 1]};
        be[r] = {cf[8 * mm + 2], cf[8 * mm + 3]};
    }
}

// R roots m .. m + R - 1 of one item (independent product chains interleaved for instruction-level
// parallelism).  R == 1 keeps the factors phi_j in registers; R > 1 recomputes them in the forward sweep
// (the registers go to the second chain instead).
template <typename T, int NW, int C, int R, bool KEEP = (R == 1)>
__device__ __forceinline__ void sym_roots(const T* cf, int m, int Mp, int lane, int warp, int t, const T (&l)[C], T (&term)[C],
                                          double& fe_acc, cplx<T> (*wtot)[2][NW], cplx<T> (&al)[R], cplx<T> (&be)[R]) {
    const cplx<T> one{(T)1, (T)0};
    const int par = (m / R) & 1;
    // 1. backward sweep: insuf_j = prod_{j' > j in chunk} phi_j'
    cplx<T> insuf[R][C], suf[R], ph1[C];
#pragma unroll
    for (int r = 0; r < R; ++r) suf[r] = one;
#pragma unroll
    for (int j = C - 1; j >= 0; --j) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const cplx<T> ph{fmaT(be[r].re, l[j], al[r].re), fmaT(be[r].im, l[j], al[r].im)};
            if (KEEP) ph1[j] = ph;
            insuf[r][j] = suf[r];
            suf[r] = cmul(suf[r], ph);
        }
    }
    // next batch's factors, requested early (latency hidden by the scan and the forward sweep)
    cplx<T> al_n[R], be_n[R];
    load_ab<T, R>(cf, m + R, Mp, al_n, be_n);
    // 2. exclusive prefix / suffix of the chunk products across the group
    cplx<T> ip[R], is[R], P[R], S[R], Q[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ip[r] = is[r] = suf[r];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const cplx<T> y = shfl_up_c(ip[r], d);
            const cplx<T> z = shfl_down_c(is[r], d);
            if (lane >= d) ip[r] = cmul(y, ip[r]);
            if (lane + d < 32) is[r] = cmul(is[r], z);
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        P[r] = shfl_up_c(ip[r], 1);
        S[r] = shfl_down_c(is[r], 1);
        if (lane == 0) P[r] = one;
        if (lane == 31) S[r] = one;
        Q[r] = shfl_c(ip[r], 31);
    }
    if (NW > 1) {
        if (lane == 31) {
#pragma unroll
            for (int r = 0; r < R; ++r) wtot[par][r][warp] = ip[r];
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < R; ++r) {
            cplx<T> Pw = one, Sw = one;
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const cplx<T> v = wtot[par][r][w];
                if (w < warp) Pw = cmul(Pw, v);
                if (w > warp) Sw = cmul(Sw, v);
            }
            Q[r] = cmul(cmul(Pw, Q[r]), Sw);
            P[r] = cmul(Pw, P[r]);
            S[r] = cmul(S[r], Sw);
        }
    }
    // 3. forward sweep: term_j += Re(A insuf_j), A = H P S prod_{j' < j} phi_j'
    cplx<T> A[R], alf[R], bef[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const cplx<T> Hm{cf[8 * (m + r) + 6], cf[8 * (m + r) + 7]};
        A[r] = cmul(cmul(Hm, P[r]), S[r]);
        alf[r] = al[r];
        bef[r] = be[r];
        if (!KEEP) { opaque(alf[r].re); opaque(alf[r].im); opaque(bef[r].re); opaque(bef[r].im); }
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            term[j] = fmaT(A[r].re, insuf[r][j].re, fmaT(-A[r].im, insuf[r][j].im, term[j]));
            const cplx<T> ph = KEEP ? ph1[j] : cplx<T>{fmaT(bef[r].re, l[j], alf[r].re), fmaT(bef[r].im, l[j], alf[r].im)};
            A[r] = cmul(A[r], ph);
        }
    }
    if (t == 0) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const T gre = cf[8 * (m + r) + 4], gim = cf[8 * (m + r) + 5];
            fe_acc += (double)gre * (double)Q[r].re - (double)gim * (double)Q[r].im;
        }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        al[r] = al_n[r];
        be[r] = be_n[r];
    }
}

// R = 0: one root per pass with the factors recomputed in the forward sweep, fewer registers (3 CTAs of
// 4 warps per SM); R = 1: factors kept in registers; R = 2: two roots per pass.
template <typename T, int NW, int C, int R>
__global__ void __launch_bounds__(32 * NW, R == 0 ? (12 / NW > 0 ? 12 / NW : 1) : (NW >= 8 ? 1 : 8 / NW))
sym_item_kernel(SymArgs<T> a, SymSplit<T> sp, int64_t s_begin) {
    extern __shared__ __align__(16) unsigned char sym_smem[];   // the signature's root table, M' x 8 T
    __shared__ cplx<T> wtot[2][2][NW];   // [root-batch parity][root in batch][warp] chunk-product totals
    __shared__ int tcnt[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = threadIdx.x;
    const int64_t item = blockIdx.x / sp.S;
    const int split = (int)(blockIdx.x - item * sp.S);
    const bool valid = true;
    const int64_t s = s_begin + item / a.B;
    const int64_t b = item - (item / a.B) * a.B;
    const SymSigDev sg = a.sigs[a.sig_of[s]];
    const int k = sg.k;
    const int64_t lo = a.off[s];
    // this CTA's roots [m0, m0 + Mps) of the item's M' (an even share when split)
    const int per = (sg.Mp + sp.S - 1) / sp.S;
    const int m0 = min(sg.Mp, split * per);
    const int Mps = min(sg.Mp, m0 + per) - m0;
    const int i0 = t * C;
    // padding literals past k get l = 1 (a certainly-False literal: p = 0), whose factor
    // alpha + beta = 1 (exactly in real arithmetic, to one rounding in the table), so the sweeps need
    // no per-literal selects; their terms are never stored
    T l[C];
    int tc = 0;
#pragma unroll
    for (int j = 0; j < C; ++j) {
        l[j] = (T)1;
        if (i0 + j < k) {
            const uint32_t w = __ldg(a.words + lo + i0 + j);
            const T xv = a.x[b * a.sb + (int64_t)(w & 0x7fffffffu) * a.sv];
            l[j] = (int)w < 0 ? -xv : xv;
            tc += (int)((xv < (T)0) != ((int)w < 0));
        }
    }
    T term[C];
#pragma unroll
    for (int j = 0; j < C; ++j) term[j] = (T)0;
    double fe_acc = 0.0;
    // root table alpha, beta, G, H (8 T per root) staged in shared memory once per item: the per-root
    // coefficient reads in the sweeps become broadcast LDS instead of dependent global loads
    T* cf = reinterpret_cast<T*>(sym_smem);   // roots m0 .. m0 + Mps - 1, indexed from 0
    {
        const T* g = a.coef + (sg.coef_off + m0) * 8;
        for (int i = t; i < Mps * 8; i += 32 * NW) cf[i] = g[i];
        __syncthreads();
    }
    const cplx<T> one{(T)1, (T)0};
    cplx<T> al[R == 0 ? 1 : R], be[R == 0 ? 1 : R];
    if (Mps > 0) load_ab<T, (R == 0 ? 1 : R)>(cf, 0, Mps, al, be);
    int m = 0;
    constexpr int RP = R == 0 ? 1 : R;   // roots per pass
    for (; m + RP <= Mps; m += RP)
        sym_roots<T, NW, C, RP, (R == 1)>(cf, m, Mps, lane, warp, t, l, term, fe_acc, wtot, al, be);
    if (R > 1 && m < Mps) {   // odd remainder: one root (al[0], be[0] hold it)
        cplx<T> al1[1] = {al[0]}, be1[1] = {be[0]};
        sym_roots<T, NW, C, 1>(cf, m, Mps, lane, warp, t, l, term, fe_acc, wtot, al1, be1);
    }
    const T wc = a.w_sym[s];
    if (sp.S > 1) {   // partials of this root share; the unsat count by split 0
        const int64_t nlit = a.off[sp.s_end] - sp.lit0;
#pragma unroll
        for (int j = 0; j < C; ++j) {
            const int i = i0 + j;
            if (i < k) {
                const uint32_t w = __ldg(a.words + lo + i);
                const T v = wc * term[j];
                sp.TbS[((int64_t)split * nlit + (lo - sp.lit0) + i) * a.B + b] = (int)w < 0 ? -v : v;
            }
        }
        if (t == 0) sp.fS[((int64_t)split * (sp.s_end - s_begin) + (s - s_begin)) * a.B + b] = fe_acc;
        if (split != 0) return;
    }
#pragma unroll
    for (int j = 0; j < C; ++j) {
        const int i = i0 + j;
        if (sp.S == 1 && i < k) {
            const uint32_t w = __ldg(a.words + lo + i);
            const T v = wc * term[j];
            a.Tb[(a.tb_fast + lo + i) * a.B + b] = (int)w < 0 ? -v : v;
        }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) tc += __shfl_xor_sync(0xffffffffu, tc, d);
    if (NW > 1) {
        if (lane == 0) tcnt[warp] = tc;
        __syncthreads();
        tc = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) tc += tcnt[w];
    }
    if (valid && t == 0) {
        if (sp.S == 1) a.fsym[s * a.B + b] = (double)wc * (sg.g0 + fe_acc);
        a.usym[s * a.B + b] = rule_sat(tc, sg.tmin, sg.tmax, sg.parity) ? 0 : 1;
    }
}

// Sum of the root-split partials of one class in split order (deterministic): the class's T rows and w (g0 +
// Re sum_m G_m Q_m) per constraint.  Grid-stride over (class literal, point) then (class constraint, point).
template <typename T>
__global__ void __launch_bounds__(256) sym_combine_kernel(SymArgs<T> a, SymSplit<T> sp, int64_t s_begin) {
    const int64_t nlit = a.off[sp.s_end] - sp.lit0, ncons = sp.s_end - s_begin;
    const int64_t nT = nlit * a.B, nF = ncons * a.B;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < nT + nF; e += (int64_t)gridDim.x * blockDim.x) {
        if (e < nT) {
            T v = sp.TbS[e];
            for (int q = 1; q < sp.S; ++q) v += sp.TbS[(int64_t)q * nT + e];
            a.Tb[(a.tb_fast + sp.lit0) * a.B + e] = v;
        } else {
            const int64_t f = e - nT;
            double v = sp.fS[f];
            for (int q = 1; q < sp.S; ++q) v += sp.fS[(int64_t)q * nF + f];
            const int64_t s = s_begin + f / a.B;
            const SymSigDev sg = a.sigs[a.sig_of[s]];
            a.fsym[s_begin * a.B + f] = (double)a.w_sym[s] * (sg.g0 + v);
        }
    }
}

// Root path for short constraints (k <= KMAX <= 32): one thread per (constraint, point) item, lanes over
// consecutive points of the same constraint (x read from x^T: coalesced), no cross-thread scan at all.  Per
// root m: backward sweep storing the in-constraint suffix products insuf_j in registers and the total Q_m,
// then the forward sweep term_j += Re(A insuf_j), A <- A phi_j (phi recomputed), A_0 = H_m.
// 14 FP lane-ops per (literal, root) and every lane busy (the warp-group kernel would idle lanes at small k).
template <typename T, int KMAX>
__global__ void __launch_bounds__(256) sym_lane_kernel(SymArgs<T> a, int64_t s_begin, int64_t n_items) {
    const int64_t item = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool valid = item < n_items;
    const int64_t it = valid ? item : n_items - 1;
    const int64_t s = s_begin + it / a.B;
    const int64_t b = it - (it / a.B) * a.B;
    const SymSigDev sg = a.sigs[a.sig_of[s]];
    const int k = sg.k;
    const int64_t lo = a.off[s];
    T l[KMAX], term[KMAX];
    int tc = 0;
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        l[j] = (T)1;      // padding literal: p = 0, factor alpha + beta = 1
        term[j] = (T)0;
        if (j < k) {
            const uint32_t w = __ldg(a.words + lo + j);
            const T xv = a.x[b * a.sb + (int64_t)(w & 0x7fffffffu) * a.sv];
            l[j] = (int)w < 0 ? -xv : xv;
            tc += (int)((xv < (T)0) != ((int)w < 0));
        }
    }
    const T* cf = a.coef + sg.coef_off * 8;
    double fe_acc = 0.0;
    for (int m = 0; m < sg.Mp; ++m) {
        const cplx<T> al{__ldg(cf + 8 * m + 0), __ldg(cf + 8 * m + 1)};
        const cplx<T> be{__ldg(cf + 8 * m + 2), __ldg(cf + 8 * m + 3)};
        cplx<T> insuf[KMAX];
        cplx<T> suf{(T)1, (T)0};
#pragma unroll
        for (int j = KMAX - 1; j >= 0; --j) {
            insuf[j] = suf;
            suf = cmul(suf, cplx<T>{fmaT(be.re, l[j], al.re), fmaT(be.im, l[j], al.im)});
        }
        cplx<T> A{__ldg(cf + 8 * m + 6), __ldg(cf + 8 * m + 7)};
#pragma unroll
        for (int j = 0; j < KMAX; ++j) {
            term[j] = fmaT(A.re, insuf[j].re, fmaT(-A.im, insuf[j].im, term[j]));
            A = cmul(A, cplx<T>{fmaT(be.re, l[j], al.re), fmaT(be.im, l[j], al.im)});
        }
        fe_acc += (double)__ldg(cf + 8 * m + 4) * (double)suf.re - (double)__ldg(cf + 8 * m + 5) * (double)suf.im;
    }
    if (!valid) return;
    const T wc = a.w_sym[s];
#pragma unroll
    for (int j = 0; j < KMAX; ++j) {
        if (j < k) {
            const uint32_t w = __ldg(a.words + lo + j);
            const T v = wc * term[j];
            a.Tb[(a.tb_fast + lo + j) * a.B + b] = (int)w < 0 ? -v : v;
        }
    }
    a.fsym[s * a.B + b] = (double)wc * (sg.g0 + fe_acc);
    a.usym[s * a.B + b] = rule_sat(tc, sg.tmin, sg.tmax, sg.parity) ? 0 : 1;
}

// ------------------------------------------------------------------------------------------------
// A7 reductions.
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

template <typename T>
struct ReduceArgs {
    int64_t B;
    int32_t n;
    int32_t n_chunks;            // tiled partial tiles (0 on the global path)
    const T* P;                  // [n_chunks][n][B]
    const T* Tb;                 // [tb_slots][B]
    const int64_t* occ_off;      // [n + 1]
    const int32_t* occ_slot;     // variable v's T rows, ascending: occ_slot[occ_off[v] .. occ_off[v + 1])
    T* grad;                     // [B][n]
    ReduceFArgs rf;              // reduce_grad_kernel<T, true>: the CTAs of variable tile 0 also reduce f / unsat
};

// block (32, 8): 32 points x 8 variables, one (variable, point) sum per thread: the chunk partials in
// chunk order, then the variable's occurrence slots in ascending order (fp64 accumulator; loads are
// issued 8 / 4 ahead but added strictly in order, so the sum order is fixed).  Output through smem so
// each point row gets 8 consecutive gradient entries.
template <typename T, bool FUSE_F>
__global__ void __launch_bounds__(256) reduce_grad_kernel(ReduceArgs<T> a) {
    __shared__ T tile[8][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t b0 = (int64_t)blockIdx.y * 32, v0 = (int64_t)blockIdx.x * 8;   // grid.x over variables (n may exceed 65535 tiles)
    const int64_t b = b0 + tx, v = v0 + ty;
    pdl_wait();      // launched programmatically after the product kernel: its partials must be complete
    pdl_trigger();
    if (FUSE_F && blockIdx.x == 0) {   // f / unsat of points b0 .. b0 + 31: warp ty sums rows ty, ty + 8, ... then in order
        __shared__ double sf[8][32];
        __shared__ int su[8][32];
        double f = 0.0;
        int u = 0;
        if (b < a.B) {
            const bool cu = a.rf.unsat != nullptr;   // the unsat partials exist only when the evaluation counted them
            for (int c = ty; c < a.rf.n_parts; c += 8) {
                f += a.rf.fpart[(int64_t)c * a.B + b];
                if (cu) u += a.rf.upart[(int64_t)c * a.B + b];
            }
            for (int64_t s = ty; s < a.rf.n_sym; s += 8) {
                f += a.rf.fsym[s * a.B + b];
                if (cu) u += a.rf.usym[s * a.B + b];
            }
        }
        sf[ty][tx] = f;
        su[ty][tx] = u;
        __syncthreads();
        if (ty == 0 && b < a.B) {
            double ft = 0.0;
            int ut = 0;
            for (int j = 0; j < 8; ++j) {
                ft += sf[j][tx];
                ut += su[j][tx];
            }
            a.rf.f[b] = ft;
            if (a.rf.unsat) a.rf.unsat[b] = ut;
        }
    }
    double acc = 0.0;
    if (v < a.n && b < a.B) {
        const int64_t stride = (int64_t)a.n * a.B;
        const T* p = a.P + v * a.B + b;
        int c = 0;
        for (; c + 8 <= a.n_chunks; c += 8) {
            T t[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) t[j] = p[(int64_t)(c + j) * stride];
#pragma unroll
            for (int j = 0; j < 8; ++j) acc += (double)t[j];
        }
        for (; c < a.n_chunks; ++c) acc += (double)p[(int64_t)c * stride];
        int64_t o = a.occ_off[v];
        const int64_t e = a.occ_off[v + 1];
        for (; o + 4 <= e; o += 4) {
            int32_t sl[4];
            T t[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) sl[j] = a.occ_slot[o + j];
#pragma unroll
            for (int j = 0; j < 4; ++j) t[j] = a.Tb[(int64_t)sl[j] * a.B + b];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc += (double)t[j];
        }
        for (; o < e; ++o) acc += (double)a.Tb[(int64_t)a.occ_slot[o] * a.B + b];
    }
    tile[ty][tx] = (T)acc;
    __syncthreads();
    const int t = ty * 32 + tx;
    const int pl = t >> 3, vl = t & 7;
    const int64_t bb = b0 + pl, vv = v0 + vl;
    if (bb < a.B && vv < a.n) a.grad[bb * a.n + vv] = tile[vl][pl];
}


// Owner-computes gradient for the short fast constraints of the global path (k <= 3, SURVEY 8(e) "owner-computes"):
// thread (variable v, point b) forms every term of v's occurrences in those constraints itself -- the constraint's
// other literals gathered from x^T (coalesced: lanes = points), the exclusive product of their factors, Prop. 1 --
// and sums them in ascending position order, then adds v's remaining T slots (long fast and root-path constraints)
// in ascending slot order (fp64 accumulation): no term round trip through HBM for the short constraints.  The
// occurrence at literal index 0 also contributes the constraint's w FE and its fused check to the tile's partial
// f / unsat row (row0 + variable tile), so every constraint is counted once.  Occurrence records are
// self-contained (the other literals' words inline) and processed four at a time with every load in flight.
// Block (32 points, 8 variables).
template <typename T>
struct OwnerArgs {
    const T* xT;                 // x^T (canonical zeros): element (v, b) at xT[(b / SB) slice_stride + v row_stride + b % SB]
    int64_t row_stride, slice_stride;   // [n][B]: B, 32 (SB = 32); 16-point slices [B/16][n][16]: 16, 16 n (SB = 16)
    int64_t B;
    int32_t n;
    const int64_t* own_off;      // [n + 1]
    const uint4* own_rec;        // {position, other word A, other word B, bucket << 8 | i << 1 | own negated}
    const FastBucketDev* buckets;
    const T* w_pos;
    const T* Tb;                 // [tb_slots][B]
    const int64_t* occ_off;      // [n + 1] the remaining (T-slot) occurrences
    const int32_t* occ_slot;
    T* grad;                     // [B][n] or null (f / unsat only)
    double* fpart;               // rows [row0 + variable tile][B]
    int32_t* upart;              // same rows, or null
    int32_t row0;
    const uint4* grp_desc;       // owner_grp_kernel: per group {record offset lo, hi, rows A, rows B}
    const int32_t* grp_var;      // slot -> variable (-1: none)
    const uint4* grp_rec;        // interleaved [row][4] records
    uint32_t grp_pitch;          // bytes per variable row of an x^T slice (8 PPT sizeof(T))
};

// L2 cache policies (createpolicy): x^T rows are gathered many times (keep them: evict_last), the occurrence records
// are read once (evict_first) -- so the streamed records do not displace x^T from L2.
__device__ __forceinline__ uint64_t l2_policy_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint4 ld_stream16(const uint4* p, uint64_t pol) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
template <typename T>
__device__ __forceinline__ T ld_keep(const T* p, uint64_t pol) {
    T v;
    if constexpr (sizeof(T) == 4) asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}

// Block = SB points x (256 / SB) variables (thread (tx = point, ty = variable)); grid (variable tiles, point slices).
template <typename T, int SB>
__global__ void __launch_bounds__(256) owner_grad_kernel(OwnerArgs<T> a) {
    constexpr int NV = 256 / SB;   // variables per block
    __shared__ T tile[NV][SB + 1];
    __shared__ double sf[NV][SB];
    __shared__ int su[NV][SB];
    const int tx = threadIdx.x % SB, ty = threadIdx.x / SB;
    const int64_t b0 = (int64_t)blockIdx.y * SB, v0 = (int64_t)blockIdx.x * NV;   // grid.x over variable tiles
    const int64_t b = b0 + tx, v = v0 + ty;
    const bool bv = b < a.B;
    const int64_t bb = bv ? b : a.B - 1;   // lanes past the batch mirror the last point (in-bounds loads, nothing stored)
    const bool want_term = a.grad != nullptr, want_unsat = a.upart != nullptr;
    double acc = 0.0, facc = 0.0;
    int uacc = 0;
    if (v < a.n) {
        const uint64_t keep = l2_policy_last(), stream = l2_policy_first();
        const T* xTb = a.xT + (bb / SB) * a.slice_stride + bb % SB;
        const T xv = ld_keep(xTb + v * a.row_stride, keep);
        int cur = -1, nch = 0;
        BucketReg<T> bk{};
        const int64_t o1 = a.own_off[v + 1];
        for (int64_t o = a.own_off[v]; o < o1; o += 4) {
            constexpr int NB = 4;
            uint4 rc[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) rc[q] = o + q < o1 ? ld_stream16(a.own_rec + o + q, stream) : make_uint4(0, 0, 0, 0);
            T xa[NB], xb[NB], wc[NB];
#pragma unroll
            for (int q = 0; q < NB; ++q) {   // every gather of the batch in flight (padding words read variable 0)
                xa[q] = ld_keep(xTb + (int64_t)(rc[q].y & 0x7fffffffu) * a.row_stride, keep);
                xb[q] = ld_keep(xTb + (int64_t)(rc[q].z & 0x7fffffffu) * a.row_stride, keep);
                wc[q] = __ldg(a.w_pos + rc[q].x);
            }
#pragma unroll
            for (int q = 0; q < NB; ++q) {
                if (o + q >= o1) break;
                const int bucket = (int)(rc[q].w >> 8), i = (int)((rc[q].w >> 1) & 3);
                if (bucket != cur) {
                    cur = bucket;
                    bk = load_bucket<T>(a.buckets + bucket);
                    nch = a.buckets[bucket].nch;
                }
                const int k = bk.k;
                const uint32_t wown = rc[q].w << 31;   // the own literal's sign bit
                T term = (T)0, fe = bk.g0;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (c >= nch) break;
                    const T ao = fmaT(flip_sign(bk.c1[c], wown), xv, bk.c0[c]);
                    const T aa = k >= 2 ? fmaT(flip_sign(bk.c1[c], rc[q].y), xa[q], bk.c0[c]) : (T)1;
                    const T ab = k >= 3 ? fmaT(flip_sign(bk.c1[c], rc[q].z), xb[q], bk.c0[c]) : (T)1;
                    const T ex = aa * ab;                                   // the other factors, in literal order
                    // all factors in literal order: own first when it is literal 0 (the only case FE is used)
                    fe = fmaT(bk.g[c], ao * ex, fe);
                    term = fmaT(bk.g[c] * flip_sign(bk.c1[c], wown), ex, term);
                }
                if (want_term) acc += (double)(wc[q] * term);
                if (i == 0) {   // the constraint's f and check, counted once (by its first literal's owner)
                    facc += (double)(wc[q] * fe);
                    if (want_unsat) {
                        uint32_t t = lit_true(xv, wown);
                        if (k >= 2) t += lit_true(xa[q], rc[q].y);
                        if (k >= 3) t += lit_true(xb[q], rc[q].z);
                        uacc += rule_sat((int)t, bk.tmin, bk.tmax, bk.parity) ? 0 : 1;
                    }
                }
            }
        }
        if (want_term) {   // the remaining occurrences' T slots, ascending (loads issued 4 ahead, added in order)
            int64_t q = a.occ_off[v];
            const int64_t e = a.occ_off[v + 1];
            for (; q + 4 <= e; q += 4) {
                int32_t sl[4];
                T t[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) sl[j] = a.occ_slot[q + j];
#pragma unroll
                for (int j = 0; j < 4; ++j) t[j] = a.Tb[(int64_t)sl[j] * a.B + bb];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc += (double)t[j];
            }
            for (; q < e; ++q) acc += (double)a.Tb[(int64_t)a.occ_slot[q] * a.B + bb];
        }
    }
    // partial f / unsat of this variable tile: variable order
    sf[ty][tx] = facc;
    su[ty][tx] = uacc;
    tile[ty][tx] = (T)acc;
    __syncthreads();
    if (ty == 0 && bv) {
        double f = 0.0;
        int u = 0;
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            f += sf[j][tx];
            u += su[j][tx];
        }
        a.fpart[((int64_t)a.row0 + blockIdx.x) * a.B + b] = f;
        if (want_unsat) a.upart[((int64_t)a.row0 + blockIdx.x) * a.B + b] = u;
    }
    if (want_term) {   // transposed write: each point row gets NV consecutive gradient entries
        const int t = threadIdx.x;
        const int pl = t / NV, vl = t % NV;
        const int64_t pb = b0 + pl, vv = v0 + vl;
        // streaming store (evict-first): the gradient is written once and must not displace the x^T slice from L2
        if (pb < a.B && vv < a.n) __stcs(a.grad + pb * a.n + vv, tile[vl][pl]);
    }
}

// PPT consecutive elements at byte offset off from base (one vector load of <= 16 bytes, read-only path).  The offset
// is a runtime product (IMAD.WIDE of the index by the row pitch: no 64-bit shift sequence).
template <typename T, int PPT>
__device__ __forceinline__ void ld_vec(const T* base, uint64_t off, T (&v)[PPT]) {
    static_assert(sizeof(T) * PPT <= 16, "vector load of at most 16 bytes");
    const char* p = reinterpret_cast<const char*>(base) + off;
    if constexpr (PPT == 1) v[0] = __ldg(reinterpret_cast<const T*>(p));
    else if constexpr (sizeof(T) == 4 && PPT == 2) {
        const float2 q = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = q.x; v[1] = q.y;
    } else if constexpr (sizeof(T) == 4 && PPT == 4) {
        const float4 q = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
        const double2 q = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = q.x; v[1] = q.y;
    }
}

// Rows [0, rows) of one owner group's section (records at rec[4 row]): the terms of this thread's variable at its PPT
// points, added in row order; FCHK (rows A: the own literal is the constraint's literal 0) also the constraint's w FE
// and its fused check.  Four rows per batch with every load in flight; the tail batch reads pad records past rows.
template <typename T, int K, int NCH, int PPT, int NB, int G, bool FCHK>
__device__ __forceinline__ void owner_grp_rows(const uint4* __restrict__ rec, int rows, const T* __restrict__ xTs, uint32_t pitch,
                                               const T* __restrict__ w_pos, const BucketReg<T>& bk, const T (&xv)[PPT],
                                               const T (&aoP)[NCH][PPT], const T (&aoN)[NCH][PPT], const T (&gP)[NCH],
                                               const T (&gN)[NCH], bool want_term, bool want_unsat, double (&acc)[PPT],
                                               double (&facc)[PPT], int (&uacc)[PPT]) {
        // software-pipelined: the next batch's records are in flight while this batch's gathers and products run (rows
    // past the section are read and masked below; the host appends pad rows past the last group)
    uint4 rc[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) rc[q] = __ldcs(rec + G * q);
    for (int j = 0; j < rows; j += NB) {
        T xa[NB][PPT], xb[NB][PPT], wc[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            if (K >= 2) ld_vec<T, PPT>(xTs, (uint64_t)(rc[q].y & 0x7fffffffu) * pitch, xa[q]);
            if (K >= 3) ld_vec<T, PPT>(xTs, (uint64_t)(rc[q].z & 0x7fffffffu) * pitch, xb[q]);
            wc[q] = __ldg(w_pos + rc[q].x);
        }
        uint4 rn[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q) rn[q] = __ldcs(rec + G * (j + NB + q));
#pragma unroll
        for (int q = 0; q < NB; ++q) {
            const bool neg = rc[q].w & 1u, pad = (rc[q].w & 2u) || j + q >= rows;
            const T w = pad ? (T)0 : wc[q];
#pragma unroll
            for (int p = 0; p < PPT; ++p) {
                T term = (T)0, fe = bk.g0;
#pragma unroll
                for (int c = 0; c < NCH; ++c) {
                    const T aa = K >= 2 ? fmaT(flip_sign(bk.c1[c], rc[q].y), xa[q][p], bk.c0[c]) : (T)1;
                    const T ab = K >= 3 ? fmaT(flip_sign(bk.c1[c], rc[q].z), xb[q][p], bk.c0[c]) : (T)1;
                    const T ex = aa * ab;
                    if (FCHK) fe = fmaT(bk.g[c], (neg ? aoN[c][p] : aoP[c][p]) * ex, fe);
                    term = fmaT(neg ? gN[c] : gP[c], ex, term);
                }
                if (want_term) acc[p] += (double)(w * term);
                if (FCHK) {
                    facc[p] += (double)(w * fe);
                    if (want_unsat) {
                        uint32_t t = lit_true(xv[p], neg ? 0x80000000u : 0u);
                        if (K >= 2) t += lit_true(xa[q][p], rc[q].y);
                        if (K >= 3) t += lit_true(xb[q][p], rc[q].z);
                        // the rule, branch-free: tmin <= t <= tmax and the parity (0 none, 1 odd, 2 even)
                        const int ti = (int)t;
                        const bool ok = ti >= bk.tmin && ti <= bk.tmax && (bk.parity == 0 || (ti & 1) == (bk.parity & 1));
                        uacc[p] += (pad || ok) ? 0 : 1;
                    }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NB; ++q) rc[q] = rn[q];
    }
}

// Owner-computes for ONE owner bucket of short constraints (k <= 3), grouped records (host.hpp grp_*): block =
// 256 / LANES variable slots x one x^T slice of SB = LANES PPT points; warp w = group w of the block (32 / LANES
// variable slots x LANES lanes), lane = PPT consecutive points (vector gathers).  The host sorts each window of 8
// blocks' variables by occurrence counts and deals it to the 8 blocks of 8 groups, padding a group's lists to its
// longest: trip counts are warp-uniform, a block's warps finish together, a record row is G = 32 / LANES records
// side by side.  The next batch of records is loaded while the current one's gathers and products run (two
// dependent misses per batch -> one).  Gradient entries are stored straight from registers (the window's blocks
// complete the rows' sectors in L2).  Per (variable, point) the order of the fp64 sum: rows A (the occurrences at
// literal index 0, which also carry the constraint's f and fused check) ascending position, rows B ascending
// position, then the variable's remaining T slots ascending -- fixed, and independent of the batch, of the slice
// width and of the point's slice position.
template <typename T, int K, int NCH, int LANES, int PPT, int WPB = 8>
__global__ void __launch_bounds__(32 * WPB, (sizeof(T) == 8 ? 2 : 3) * 8 / WPB) owner_grp_kernel(OwnerArgs<T> a, int32_t bucket) {
    constexpr int SB = LANES * PPT;          // points per x^T slice
    constexpr int G = 32 / LANES;            // variable slots per warp (= group)
    constexpr int NS = WPB * G;              // variable slots per block (WPB warps = groups)
    constexpr int NB = PPT == 4 ? 2 : 4;     // record rows per batch (registers: 80 at 4 points per thread)
    static_assert(LANES * PPT >= 1 && 32 % LANES == 0, "lanes divide a warp");
    __shared__ double sf[NS][SB];
    __shared__ int su[NS][SB];
    const int t = threadIdx.x, lane = t % LANES, slot = t / LANES;
    const int64_t v0 = (int64_t)blockIdx.x * NS, b0 = (int64_t)blockIdx.y * SB;
    const bool want_term = a.grad != nullptr, want_unsat = a.upart != nullptr;
    const BucketReg<T> bk = load_bucket<T>(a.buckets + bucket);
    const int32_t v = a.grp_var[v0 + slot];
    const T* xTs = a.xT + (int64_t)blockIdx.y * SB * a.n + lane * PPT;
    double acc[PPT], facc[PPT];
    int uacc[PPT];
#pragma unroll
    for (int p = 0; p < PPT; ++p) { acc[p] = 0.0; facc[p] = 0.0; uacc[p] = 0; }
    T xv[PPT];
    const uint32_t pitch = a.grp_pitch;   // = SB * sizeof(T), a runtime value
    ld_vec<T, PPT>(xTs, (uint64_t)(v < 0 ? 0 : v) * pitch, xv);
    T aoP[NCH][PPT], aoN[NCH][PPT], gP[NCH], gN[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        gP[c] = bk.g[c] * bk.c1[c];
        gN[c] = bk.g[c] * -bk.c1[c];
#pragma unroll
        for (int p = 0; p < PPT; ++p) {
            aoP[c][p] = fmaT(bk.c1[c], xv[p], bk.c0[c]);
            aoN[c][p] = fmaT(-bk.c1[c], xv[p], bk.c0[c]);
        }
    }
    const uint4 d = a.grp_desc[blockIdx.x * WPB + t / 32];
    const uint4* rec = a.grp_rec + (((int64_t)d.y << 32) | d.x) + slot % G;   // record row 0 of the group, this slot
    owner_grp_rows<T, K, NCH, PPT, NB, G, true>(rec, (int)d.z, xTs, pitch, a.w_pos, bk, xv, aoP, aoN, gP, gN, want_term,
                                                want_unsat, acc, facc, uacc);
    owner_grp_rows<T, K, NCH, PPT, NB, G, false>(rec + G * (int64_t)d.z, (int)d.w, xTs, pitch, a.w_pos, bk, xv, aoP, aoN,
                                                 gP, gN, want_term, want_unsat, acc, facc, uacc);
    if (want_term && v >= 0) {   // the variable's remaining T slots (long fast / root-path constraints), ascending
        const int64_t e = a.occ_off[v + 1];
        for (int64_t q = a.occ_off[v]; q < e; ++q) {
            const int64_t sl = a.occ_slot[q];
#pragma unroll
            for (int p = 0; p < PPT; ++p) {
                const int64_t bb = min(b0 + lane * PPT + p, a.B - 1);
                acc[p] += (double)a.Tb[sl * a.B + bb];
            }
        }
    }
#pragma unroll
    for (int p = 0; p < PPT; ++p) {
        sf[slot][lane * PPT + p] = facc[p];
        su[slot][lane * PPT + p] = uacc[p];
        // the gradient entry straight from the register (the block's variables are scattered over its window: the
        // window's 8 blocks, launched together, complete the rows' sectors in L2)
        const int64_t pb = b0 + lane * PPT + p;
        if (want_term && v >= 0 && pb < a.B) __stcs(a.grad + pb * a.n + v, (T)acc[p]);
    }
    __syncthreads();
    if (t < SB && b0 + t < a.B) {   // partial f / unsat of this block, slot order
        double f = 0.0;
        int u = 0;
#pragma unroll 8
        for (int j = 0; j < NS; ++j) {
            f += sf[j][t];
            u += su[j][t];
        }
        a.fpart[((int64_t)a.row0 + blockIdx.x) * a.B + b0 + t] = f;
        if (want_unsat) a.upart[((int64_t)a.row0 + blockIdx.x) * a.B + b0 + t] = u;
    }
}

// Fold partial rows [src, src + nrows) into rows [dst, dst + ceil(nrows / 256)): group g = rows 256 g .. 256 g + 255,
// warp w sums its rows w, w + 8, ... in ascending order, then the 8 warp sums in warp order (a fixed tree: the f /
// unsat totals stay deterministic for any batch).  grid (groups, point tiles), block 256.
template <int NW>   // NW = 8 (a template so that every translation unit may include this header)
__global__ void __launch_bounds__(32 * NW) fold_rows_kernel(double* fpart, int32_t* upart, int64_t B, int64_t src, int64_t nrows,
                                                        int64_t dst) {
    __shared__ double sf[8][32];
    __shared__ int su[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.y * 32 + lane;
    const int64_t r0 = (int64_t)blockIdx.x * 256, r1 = min(nrows, r0 + 256);
    double f = 0.0;
    int u = 0;
    if (b < B)
        for (int64_t r = r0 + w; r < r1; r += 8) {
            f += fpart[(src + r) * B + b];
            if (upart) u += upart[(src + r) * B + b];
        }
    sf[w][lane] = f;
    su[w][lane] = u;
    __syncthreads();
    if (w == 0 && b < B) {
        double t = 0.0;
        int tu = 0;
        for (int j = 0; j < 8; ++j) {
            t += sf[j][lane];
            tu += su[j][lane];
        }
        fpart[(dst + blockIdx.x) * B + b] = t;
        if (upart) upart[(dst + blockIdx.x) * B + b] = tu;
    }
}

// ---- reductions of POINT-major partials (the TMEM kernel writes P[chunk][b][v]): one warp per point, lanes over
//      variables.  Sums in the same fixed orders as reduce_grad_kernel / reduce_f_kernel (so the result bits do not
//      depend on which kernel reduced them): gradient = chunk partials in chunk order, then the variable's T slots
//      ascending (fp64); f / unsat = `groups` interleaved row groups (rows j, j + groups, ... of the chunk partials,
//      then of the root-path constraints), groups added in order.
template <typename T>
struct PmReduce {
    int64_t B;
    int32_t n, n_chunks, groups;
    int64_t n_sym;
    const T* P;                  // [n_chunks][B][n]
    const T* Tb;                 // [tb_slots][B]
    const int64_t* occ_off;
    const int32_t* occ_slot;
    const double* fpart;         // [n_chunks][B]
    const int32_t* upart;        // or null (no check)
    const double* fsym;          // [n_sym][B]
    const int32_t* usym;
};

template <typename T>
__device__ __forceinline__ double pm_grad(const PmReduce<T>& a, int64_t b, int v) {
    double acc = 0.0;
    const T* p = a.P + b * a.n + v;
    const int64_t stride = a.B * a.n;
    int c = 0;
    for (; c + 4 <= a.n_chunks; c += 4) {
        T t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = p[(int64_t)(c + j) * stride];
#pragma unroll
        for (int j = 0; j < 4; ++j) acc += (double)t[j];
    }
    for (; c < a.n_chunks; ++c) acc += (double)p[(int64_t)c * stride];
    for (int64_t o = a.occ_off[v]; o < a.occ_off[v + 1]; ++o) acc += (double)a.Tb[(int64_t)a.occ_slot[o] * a.B + b];
    return acc;
}

// f / unsat of point b by one whole warp: lane j < groups sums group j (chunk rows j, j + groups, ... then root-path
// rows j, j + groups, ..., ascending), then the group sums are added in group order (moved by shuffles) -- the order
// of reduce_f_kernel, bit for bit.  Every lane returns the result.
template <typename T>
__device__ __forceinline__ double pm_f_warp(const PmReduce<T>& a, int64_t b, int* unsat) {
    const int lane = threadIdx.x & 31;
    double fj = 0.0;
    int u = 0;
    if (lane < a.groups) {
        for (int c = lane; c < a.n_chunks; c += a.groups) {
            fj += a.fpart[(int64_t)c * a.B + b];
            if (a.upart) u += a.upart[(int64_t)c * a.B + b];
        }
        for (int64_t s = lane; s < a.n_sym; s += a.groups) {
            fj += a.fsym[s * a.B + b];
            if (a.upart) u += a.usym[s * a.B + b];
        }
    }
    double f = 0.0;
    for (int j = 0; j < a.groups; ++j) f += __shfl_sync(0xffffffffu, fj, j);
    *unsat = __reduce_add_sync(0xffffffffu, u);
    return f;
}

// grad [B][n] (or null), f [B], unsat [B] (or null): one CTA per point, one thread per variable (n <= 256 on the TMEM
// path; blockDim = n rounded up to a warp), so every partial of the point is loaded in one round trip.
template <typename T>
__global__ void __launch_bounds__(256) reduce_pm_kernel(PmReduce<T> a, T* grad, double* f, int32_t* unsat) {
    pdl_wait();
    const int64_t b = blockIdx.x;
    if (grad)
        for (int v = threadIdx.x; v < a.n; v += blockDim.x) grad[b * a.n + v] = (T)pm_grad(a, b, v);
    if (threadIdx.x < 32) {
        int u = 0;
        const double fb = pm_f_warp(a, b, &u);
        if (threadIdx.x == 0) {
            f[b] = fb;
            if (unsat) unsat[b] = u;
        }
    }
}

// one CTA (32 NWF threads) per 32 points: lane = point, warp w sums rows w, w + NWF, ... in ascending
// order, then the NWF warp sums are added in warp order -- a fixed summation order for a given launch
// shape (deterministic, no atomics).  NWF = 32 when few point tiles must cover many partial rows.
template <int NWF>
__global__ void __launch_bounds__(32 * NWF) reduce_f_kernel(ReduceFArgs a) {
    __shared__ double sf[NWF][32];
    __shared__ int su[NWF][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t b = (int64_t)blockIdx.x * 32 + lane;
    double f = 0.0;
    int u = 0;
    if (b < a.B) {
        const bool cu = a.unsat != nullptr;   // the unsat partials exist only when the evaluation counted them
        // rows w, w + NWF, ...: loads issued 8 at a time (one latency per batch), added strictly in row order
        int c = w;
        for (; c + 7 * NWF < a.n_parts; c += 8 * NWF) {
            double fv[8];
            int uv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                fv[j] = a.fpart[(int64_t)(c + j * NWF) * a.B + b];
                uv[j] = cu ? a.upart[(int64_t)(c + j * NWF) * a.B + b] : 0;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                f += fv[j];
                u += uv[j];
            }
        }
        for (; c < a.n_parts; c += NWF) {
            f += a.fpart[(int64_t)c * a.B + b];
            if (cu) u += a.upart[(int64_t)c * a.B + b];
        }
        for (int64_t s = w; s < a.n_sym; s += NWF) {
            f += a.fsym[s * a.B + b];
            if (cu) u += a.usym[s * a.B + b];
        }
    }
    sf[w][lane] = f;
    su[w][lane] = u;
    __syncthreads();
    if (w == 0 && b < a.B) {
        double ft = 0.0;
        int ut = 0;
        for (int j = 0; j < NWF; ++j) {
            ft += sf[j][lane];
            ut += su[j][lane];
        }
        a.f[b] = ft;
        if (a.unsat) a.unsat[b] = ut;
    }
}

// x^T in 1-point slices is x itself: a canonicalising copy (-0.0 -> +0.0, as transpose_kernel does), 16 bytes per
// thread per step, grid-stride.
template <typename T>
__global__ void __launch_bounds__(256) canon_copy_kernel(const T* __restrict__ x, T* __restrict__ y, int64_t count) {
    constexpr int V = 16 / sizeof(T);
    const bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;   // (a view)
    const int64_t nv = aligned ? count / V : 0, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
        if constexpr (sizeof(T) == 4) {
            float4 q = reinterpret_cast<const float4*>(x)[i];
            q.x += 0.0f; q.y += 0.0f; q.z += 0.0f; q.w += 0.0f;
            reinterpret_cast<float4*>(y)[i] = q;
        } else {
            double2 q = reinterpret_cast<const double2*>(x)[i];
            q.x += 0.0; q.y += 0.0;
            reinterpret_cast<double2*>(y)[i] = q;
        }
    }
    for (int64_t i = nv * V + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) y[i] = x[i] + (T)0;
}

// x [B][n] -> x^T: W = 0 [n][B]; W > 0: W-point slices [B/W][n][W] (each slice contiguous).
template <typename T, int W = 0>
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
        if (b < B && v < n) {
            const int64_t o = W > 0 ? (b / W) * W * (int64_t)n + v * W + (b % W) : v * B + b;
            xT[o] = tile[tx][ty + 8 * j] + (T)0;   // + 0: canonical zeros (-0.0 -> +0.0)
        }
    }
}

}  // namespace dev
}  // namespace ffsat
