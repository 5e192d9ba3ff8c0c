// kernels_solve.cuh -- sm_100a kernels of the CLS loop (steps A8-A10 of DESIGN.md).
//
//   init_points_kernel     Alg. 1 line 1: x0 uniform in [-1,1]^n, Philox4x32-10 keyed by
//                          (seed, global point, round) so trajectories do not depend on the GPU count.
//   pgd_step_kernel        Alg. 4: Armijo accept/reject of the trial point just evaluated,
//                          eta update, convergence (eta < eta_min), solved-trial capture, then
//                          the next trial x' = clip(x - eta g, -1, 1) and <g, x' - x>; one CTA per point.
//   check_kernel           Alg. 1 line 5 / Thm. 4: exact integer check of sgn(x) per
//                          (constraint, point): unsat[b] and U[c].
//   erwa_kernel            Prop. 3: w <- (1-alpha) w + alpha U/max U (skipped if max U = 0).
//   rephase_kernel         O / F / R phases in the policy cycle, offset by global point.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels_common.cuh"

namespace ffsat {
namespace dev {

// Philox4x32-10 (Salmon et al., SC'11)
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k.x += W0;
            k.y += W1;
        }
        uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
        uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// value i of the (seed, point, round) stream, in (-1, 1), exactly representable in fp32
__device__ __forceinline__ double philox_pm1(uint64_t seed, uint32_t point, uint32_t rnd, uint32_t i) {
    uint4 o = philox4x32_10(make_uint4(i >> 2, point, rnd, 0x51A7u), make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
    uint32_t w = (i & 3) == 0 ? o.x : (i & 3) == 1 ? o.y : (i & 3) == 2 ? o.z : o.w;
    return ((double)(w >> 8) + 0.5) * (1.0 / 8388608.0) - 1.0;
}

template <typename T>
__global__ void init_points_kernel(T* x, int64_t B, int32_t n, uint64_t seed, int64_t point0, uint32_t rnd) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * n) return;
    const int64_t b = idx / n;
    const int32_t v = (int32_t)(idx - b * n);
    x[idx] = (T)philox_pm1(seed, (uint32_t)(point0 + b), rnd, (uint32_t)v);
}

struct PgdArgs {
    int64_t B;
    int32_t n;
    double eta0, eta_min, c1;
    int32_t max_inner;
    void* X;        // [B][n] accepted
    void* Xp;       // [B][n] trial
    void* Gx;       // [B][n] grad at X
    void* Gp;       // [B][n] grad at trial
    double* fX;
    double* fP;
    double* dot;    // <Gx, Xp - X>
    double* eta;
    int32_t* done;
    int32_t* iters;
    int32_t* unsatP;   // falsified count of sgn(trial) from the fused check of the trial eval
    int32_t* solved;   // per point: 1 once a trial satisfied everything
    int8_t* sol;       // [B][n] the first satisfying trial's assignment (-1 True / +1 False)
    int32_t mode;      // 0 = propose only (round start), 1 = accept then propose
};

// one CTA (256 threads) per point
template <typename T>
__global__ void __launch_bounds__(256) pgd_step_kernel(PgdArgs a) {
    __shared__ double red[256];
    __shared__ int s_acc;
    const int64_t b = blockIdx.x;
    const int n = a.n;
    T* X = reinterpret_cast<T*>(a.X) + b * n;
    T* Xp = reinterpret_cast<T*>(a.Xp) + b * n;
    T* Gx = reinterpret_cast<T*>(a.Gx) + b * n;
    const T* Gp = reinterpret_cast<const T*>(a.Gp) + b * n;
    int8_t* sol = a.sol + b * n;
    if (a.mode == 0) {
        // round start: the evaluated point is x itself
        if (threadIdx.x == 0) {
            int newly = (a.unsatP[b] == 0 && !a.solved[b]) ? 1 : 0;
            if (newly) a.solved[b] = 1;
            s_acc = newly << 1;
        }
        __syncthreads();
        if (s_acc & 2)
            for (int v = threadIdx.x; v < n; v += blockDim.x) sol[v] = X[v] < (T)0 ? (int8_t)-1 : (int8_t)1;
    }
    if (a.mode == 1) {
        if (threadIdx.x == 0) {
            int acc = 0;
            if (!a.done[b]) {
                acc = a.fP[b] <= a.fX[b] + a.c1 * a.dot[b];
                double eta = a.eta[b];
                eta = acc ? fmin(2.0 * eta, a.eta0) : 0.5 * eta;
                a.eta[b] = eta;
                int it = a.iters[b] + 1;
                a.iters[b] = it;
                if (acc) a.fX[b] = a.fP[b];
                if (eta < a.eta_min || it >= a.max_inner) a.done[b] = 1;
            }
            // any trial whose rounded assignment satisfies every constraint is a solution (Thm. 4)
            int newly = (a.unsatP[b] == 0 && !a.solved[b]) ? 1 : 0;
            if (newly) a.solved[b] = 1;
            s_acc = acc | (newly << 1);
        }
        __syncthreads();
        const int flags = s_acc;
        if (flags & 2)
            for (int v = threadIdx.x; v < n; v += blockDim.x) sol[v] = Xp[v] < (T)0 ? (int8_t)-1 : (int8_t)1;
        if (flags & 1)
            for (int v = threadIdx.x; v < n; v += blockDim.x) {
                X[v] = Xp[v];
                Gx[v] = Gp[v];
            }
    }
    // next trial point
    const bool act = !a.done[b];
    const T eta = (T)a.eta[b];
    double d = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        T xv = X[v];
        T g = Gx[v];
        T xn = act ? clamp1(xv - eta * g) : xv;
        Xp[v] = xn;
        d += (double)g * (double)(xn - xv);
    }
    red[threadIdx.x] = d;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) a.dot[b] = red[0];
}

// sgn(x) check (Alg. 1 line 5): exact integer count t of True literals per (constraint, point).
// CTA = 32 points (lane = point) x a contiguous range of constraints (warp = constraint).  The point
// values come from a shared-memory tile [n][33] (SMEM = true, small n) or from the transposed copy
// xT [n][B] (coalesced 128-byte rows, large n).  U[c] += #points of this tile falsifying c (warp ballot +
// popc, one integer atomic per warp-constraint); unsat[b] += this CTA's count (one integer atomic per
// point).  Integer atomics: the totals are exact and order-independent.  U and unsat are zeroed before.
struct CheckArgs {
    const void* X;      // [B][n] (SMEM) or xT [n][B]
    int64_t B;
    int32_t n;
    int64_t m;
    int64_t cons_per_cta;
    const int64_t* off;       // [m + 1] position-order literal offsets into words
    const uint32_t* words;    // var | neg << 31
    const int32_t* rule;      // [m][3]
    int32_t* U;               // [m]
    int32_t* unsat;           // [B]
};

__device__ __forceinline__ uint32_t sign_xor(float xv, uint32_t w) { return (__float_as_uint(xv) ^ w) >> 31; }
__device__ __forceinline__ uint32_t sign_xor(double xv, uint32_t w) { return ((uint32_t)__double2hiint(xv) ^ w) >> 31; }

template <typename T, bool SMEM>
__global__ void __launch_bounds__(256) check_kernel(CheckArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int ucnt[8][32];
    const T* X = reinterpret_cast<const T*>(a.X);
    T* xs = reinterpret_cast<T*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * 32, b = b0 + lane;
    const bool bv = b < a.B;
    if (SMEM) {   // x tile, 8 independent loads in flight per thread
        const int tot = 32 * a.n;
        for (int base = 0; base < tot; base += 8 * 256) {
            T v8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                const int r = idx / a.n, v = idx - r * a.n;
                v8[q] = (idx < tot && b0 + r < a.B) ? __ldg(X + (b0 + r) * a.n + v) : (T)0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                if (idx < tot) {
                    const int r = idx / a.n, v = idx - r * a.n;
                    xs[v * 33 + r] = v8[q];
                }
            }
        }
        __syncthreads();
    }
    const int64_t c0 = (int64_t)blockIdx.y * a.cons_per_cta;
    const int64_t c1 = min(a.m, c0 + a.cons_per_cta);
    int mine = 0;
    for (int64_t c = c0 + warp; c < c1; c += 8) {
        const int64_t lo = a.off[c], hi = a.off[c + 1];
        int t = 0;
        int64_t i = lo;
        for (; i + 4 <= hi; i += 4) {           // four literals' loads in flight
            uint32_t w[4];
            T xv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) w[q] = __ldg(a.words + i + q);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t v = w[q] & 0x7fffffffu;
                xv[q] = SMEM ? xs[v * 33 + lane] : (bv ? X[(int64_t)v * a.B + b] : (T)0);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) t += (int)((xv[q] < (T)0) != ((int)w[q] < 0));
        }
        for (; i < hi; ++i) {
            const uint32_t w = __ldg(a.words + i);
            const uint32_t v = w & 0x7fffffffu;
            const T xv = SMEM ? xs[v * 33 + lane] : (bv ? X[(int64_t)v * a.B + b] : (T)0);
            t += (int)((xv < (T)0) != ((int)w < 0));
        }
        const bool uns = bv && !rule_sat(t, a.rule[3 * c], a.rule[3 * c + 1], a.rule[3 * c + 2]);
        mine += uns ? 1 : 0;
        const int cnt = __popc(__ballot_sync(0xffffffffu, uns));
        if (lane == 0 && cnt) atomicAdd(a.U + c, cnt);
    }
    ucnt[warp][lane] = mine;
    __syncthreads();
    if (warp == 0 && bv) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) tot += ucnt[w][lane];
        if (tot) atomicAdd(a.unsat + b, tot);
    }
}

// Same check when every constraint has the same length K <= 16 and n fits the smem tile (the uniform k-SAT
// case): CSR offsets are c K, the K literal words are read as uniform loads, and the True-literal count uses
// the sign bit of the (canonical-zero) tile value: one LDS, one LOP3 and one LEA.HI per literal.
template <typename T, int K>
__global__ void __launch_bounds__(256) check_uniform_kernel(CheckArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ int ucnt[8][32];
    const T* X = reinterpret_cast<const T*>(a.X);
    T* xs = reinterpret_cast<T*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t b0 = (int64_t)blockIdx.x * 32, b = b0 + lane;
    const bool bv = b < a.B;
    {
        const int tot = 32 * a.n;
        for (int base = 0; base < tot; base += 8 * 256) {
            T v8[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                const int r = idx / a.n, v = idx - r * a.n;
                v8[q] = (idx < tot && b0 + r < a.B) ? __ldg(X + (b0 + r) * a.n + v) : (T)0;
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int idx = base + q * 256 + (int)threadIdx.x;
                if (idx < tot) {
                    const int r = idx / a.n, v = idx - r * a.n;
                    xs[v * 33 + r] = v8[q] + (T)0;   // canonical zero: the sign bit is exactly x < 0
                }
            }
        }
        __syncthreads();
    }
    const int c0 = (int)((int64_t)blockIdx.y * a.cons_per_cta);
    const int c1 = (int)min(a.m, (int64_t)c0 + a.cons_per_cta);
    const T* xl = xs + lane;
    int mine = 0;
    for (int c = c0 + warp; c < c1; c += 8) {
        uint32_t w[K];
#pragma unroll
        for (int i = 0; i < K; ++i) w[i] = __ldg(a.words + c * K + i);
        uint32_t t = 0;
#pragma unroll
        for (int i = 0; i < K; ++i) {
            const T xv = xl[(w[i] & 0x7fffffffu) * 33];
            t += sign_xor(xv, w[i]);
        }
        const bool uns = bv && !rule_sat((int)t, __ldg(a.rule + 3 * c), __ldg(a.rule + 3 * c + 1), __ldg(a.rule + 3 * c + 2));
        mine += uns ? 1 : 0;
        const int cnt = __popc(__ballot_sync(0xffffffffu, uns));
        if (lane == 0 && cnt) atomicAdd(a.U + c, cnt);
    }
    ucnt[warp][lane] = mine;
    __syncthreads();
    if (warp == 0 && bv) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) tot += ucnt[w][lane];
        if (tot) atomicAdd(a.unsat + b, tot);
    }
}

// X [B][n] -> xT [n][B] for the large-n check (32 x 32 tiles through smem)
template <typename T>
__global__ void __launch_bounds__(256) transpose_search_kernel(const T* __restrict__ x, T* __restrict__ xT, int64_t B, int32_t n) {
    __shared__ T tile[32][33];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const int64_t v0 = (int64_t)blockIdx.x * 32, b0 = (int64_t)blockIdx.y * 32;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t bb = b0 + ty + 8 * j, v = v0 + tx;
        if (bb < B && v < n) tile[ty + 8 * j][tx] = x[bb * n + v];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int64_t v = v0 + ty + 8 * j, bb = b0 + tx;
        if (bb < B && v < n) xT[v * B + bb] = tile[tx][ty + 8 * j];
    }
}

// ERWA (single block): maxU, then w = (1 - alpha) w + alpha U / maxU
template <typename T>
__global__ void __launch_bounds__(1024) erwa_kernel(T* w, const int32_t* U, int64_t m, double alpha) {
    __shared__ int red[1024];
    int mx = 0;
    for (int64_t c = threadIdx.x; c < m; c += blockDim.x) mx = max(mx, U[c]);
    red[threadIdx.x] = mx;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] = max(red[threadIdx.x], red[threadIdx.x + s]);
        __syncthreads();
    }
    mx = red[0];
    if (mx == 0) return;
    const double inv = 1.0 / (double)mx;
    for (int64_t c = threadIdx.x; c < m; c += blockDim.x)
        w[c] = (T)((1.0 - alpha) * (double)w[c] + alpha * ((double)U[c] * inv));
}

// policy codes: 'R' = 0, 'O' = 1, 'F' = 2 per cycle position
template <typename T>
__global__ void rephase_kernel(T* x, int64_t B, int32_t n, uint64_t seed, int64_t point0, uint32_t new_round,
                               int32_t cycle_len, int32_t p0, int32_t p1, int32_t p2) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * n) return;
    const int64_t b = idx / n;
    const int32_t v = (int32_t)(idx - b * n);
    const int64_t gb = point0 + b;
    const int ph_i = (int)(((int64_t)new_round - 1 + gb) % cycle_len);
    const int ph = ph_i == 0 ? p0 : ph_i == 1 ? p1 : p2;
    if (ph == 2) x[idx] = -x[idx];
    else if (ph == 0) x[idx] = (T)philox_pm1(seed, (uint32_t)gb, new_round, (uint32_t)v);
}

__global__ void reset_round_kernel(double* eta, int32_t* done, int32_t* iters, int64_t B, double eta0) {
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    eta[b] = eta0;
    done[b] = 0;
    iters[b] = 0;
}

// stats: active count, lowest solved index, min unsat and its lowest index (single block)
__global__ void __launch_bounds__(1024) stats_kernel(const int32_t* done, const int32_t* solved, const int32_t* unsat,
                                                     int64_t B, int64_t* out /* [4] */) {
    __shared__ long long s_act[1024], s_sol[1024], s_best[1024];
    long long act = 0, sol = INT64_MAX, best = INT64_MAX;  // best packs (unsat << 32) | index
    for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
        act += done[b] ? 0 : 1;
        if (solved[b] && b < sol) sol = b;
        long long key = ((long long)unsat[b] << 32) | (long long)b;
        if (key < best) best = key;
    }
    s_act[threadIdx.x] = act;
    s_sol[threadIdx.x] = sol;
    s_best[threadIdx.x] = best;
    __syncthreads();
    for (int s = 512; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) {
            s_act[threadIdx.x] += s_act[threadIdx.x + s];
            s_sol[threadIdx.x] = min(s_sol[threadIdx.x], s_sol[threadIdx.x + s]);
            s_best[threadIdx.x] = min(s_best[threadIdx.x], s_best[threadIdx.x + s]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = s_act[0];
        out[1] = s_sol[0] == INT64_MAX ? -1 : s_sol[0];
        out[2] = s_best[0] == INT64_MAX ? -1 : (s_best[0] >> 32);
        out[3] = s_best[0] == INT64_MAX ? -1 : (s_best[0] & 0xffffffffLL);
    }
}

template <typename T>
__global__ void permute_weights_kernel(T* w_pos, const double* w_orig, const int64_t* order, int64_t m) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < m) w_pos[p] = (T)w_orig[order[p]];
}

template <typename T>
__global__ void unpermute_weights_kernel(double* w_orig, const T* w_pos, const int64_t* order, int64_t m) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p < m) w_orig[order[p]] = (double)w_pos[p];
}

}  // namespace dev
}  // namespace ffsat
