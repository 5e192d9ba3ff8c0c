// kernels_solve.cuh -- sm_100a kernels of the CLS loop (steps A8-A10 of DESIGN.md).
//
//   init_points_kernel     Alg. 1 line 1: x0 uniform in [-1,1]^n, Philox4x32-10 keyed by
//                          (seed, global point, round) so trajectories do not depend on the GPU count.
//   pgd_step_kernel        Alg. 4: Armijo accept/reject of the trial point just evaluated,
//                          eta update, convergence (eta < eta_min), solved-trial capture, then
//                          the next trial x' = clip(x - eta g, -1, 1) and <g, x' - x>; one CTA per point.
//   signpack_kernel,       Alg. 1 line 5 / Thm. 4: exact integer check of sgn(x) per
//   check_bits_kernel      (constraint, point) on sign words of 32 points: unsat[b] and U[c].
//                          Integer atomics only: totals are exact and order-independent.
//   umax_kernel,           Prop. 3: w <- (1-alpha) w + alpha U/max U (skipped if max U = 0).
//   erwa_kernel
//   rephase_kernel         O / F / R phases in the policy cycle, offset by global point.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels_common.cuh"
#include "kernels_eval.cuh"

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
    int32_t checked;   // 1: unsatP holds the fused check of the evaluated point (check iterations only)
};

// one CTA (256 threads) per point.  The point's search state is loaded first (one latency), the decision is thread 0's,
// then one pass over the point's row: accept (x <- x', g <- g') and the next trial x'' = clip(x - eta g) with
// <g, x'' - x> (warp sums, then the warp sums in order: a fixed order).
// NT threads per CTA (a function of n only, so a point's bits never depend on the batch: 1024 for n >= 2048)
template <typename T, int NT = 256>
__global__ void __launch_bounds__(NT) pgd_step_kernel(PgdArgs a) {
    pdl_wait();   // launched programmatically after the gradient reduction
    __shared__ double s_red[NT / 32];
    __shared__ int s_acc, s_done;
    __shared__ double s_eta;
    const int64_t b = blockIdx.x;
    const int n = a.n;
    T* X = reinterpret_cast<T*>(a.X) + b * n;
    T* Xp = reinterpret_cast<T*>(a.Xp) + b * n;
    T* Gx = reinterpret_cast<T*>(a.Gx) + b * n;
    const T* Gp = reinterpret_cast<const T*>(a.Gp) + b * n;
    int8_t* sol = a.sol + b * n;
    if (threadIdx.x == 0) {
        const double fX = a.fX[b], fP = a.fP[b], dot = a.dot[b];
        double eta = a.eta[b];
        int done = a.done[b], iters = a.iters[b];
        const int unsatP = a.unsatP[b], solved = a.solved[b];
        int acc = 0;
        if (a.mode == 0) {   // round start: the evaluated point is x itself; eta, done, iteration count restart
            eta = a.eta0;
            done = 0;
            a.iters[b] = 0;
        } else if (!done) {
            acc = fP <= fX + a.c1 * dot;
            eta = acc ? fmin(2.0 * eta, a.eta0) : 0.5 * eta;
            const int it = iters + 1;
            a.iters[b] = it;
            if (acc) a.fX[b] = fP;
            if (eta < a.eta_min || it >= a.max_inner) done = 1;
        }
        a.eta[b] = eta;
        a.done[b] = done;
        // any checked trial whose rounded assignment satisfies every constraint is a solution (Thm. 4)
        const int newly = (a.checked && unsatP == 0 && !solved) ? 1 : 0;
        if (newly) a.solved[b] = 1;
        s_acc = acc | (newly << 1);
        s_eta = eta;
        s_done = done;
    }
    __syncthreads();
    const int flags = s_acc;
    const bool act = !s_done;
    const T eta = (T)s_eta;
    double d = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        T xv, g;
        if (a.mode == 1 && (flags & 1)) {
            xv = Xp[v];
            g = Gp[v];
            X[v] = xv;
            Gx[v] = g;
        } else {
            xv = X[v];
            g = Gx[v];
        }
        if (flags & 2) sol[v] = (a.mode == 0 ? xv : Xp[v]) < (T)0 ? (int8_t)-1 : (int8_t)1;
        const T xn = act ? clamp1(xv - eta * g) : xv;
        Xp[v] = xn;
        d += (double)g * (double)(xn - xv);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
        a.dot[b] = t;
    }
}

// The PGD step fused with the reduction of point-major partials (tiled TMEM path, n <= 256 <= blockDim): per point
// b the CTA sums its gradient (one variable per thread) and f / unsat from the evaluation's partials in the fixed
// orders of reduce_pm_kernel (the same bits), then takes the Armijo decision and proposes the next trial exactly as
// pgd_step_kernel -- the gradient of the trial never round-trips through HBM.  mode 0 (round start): the evaluated
// point is x itself (f and gradient at x, first trial).  One CTA per point.
template <typename T>
__global__ void __launch_bounds__(256) pgd_fused_kernel(PgdArgs a, PmReduce<T> r) {
    pdl_wait();
    __shared__ double s_red[8];
    __shared__ int s_acc, s_done;
    __shared__ double s_f, s_eta;
    __shared__ int s_u;
    const int64_t b = blockIdx.x;
    const int n = a.n;
    const int v = threadIdx.x;
    T* X = reinterpret_cast<T*>(a.X) + b * n;
    T* Xp = reinterpret_cast<T*>(a.Xp) + b * n;
    T* Gx = reinterpret_cast<T*>(a.Gx) + b * n;
    int8_t* sol = a.sol + b * n;
    // every load of the step first (they are independent, so one memory latency instead of a chain): the point's
    // rows, the search state of the point, its partials
    T x0 = (T)0, xp0 = (T)0, g0 = (T)0;
    if (v < n) {
        x0 = X[v];
        if (a.mode != 0) xp0 = Xp[v];
        g0 = Gx[v];
    }
    double st_fX = 0.0, st_dot = 0.0, st_eta = 0.0;
    int st_done = 0, st_iters = 0, st_solved = 0;
    if (threadIdx.x == 0) {
        st_fX = a.fX[b]; st_dot = a.dot[b]; st_eta = a.eta[b];
        st_done = a.done[b]; st_iters = a.iters[b]; st_solved = a.solved[b];
    }
    const T g = v < n ? (T)pm_grad(r, b, v) : (T)0;   // gradient at the evaluated point
    if (threadIdx.x < 32) {
        int u = 0;
        const double fb = pm_f_warp(r, b, &u);
        if (threadIdx.x == 0) {
            s_f = fb;
            s_u = u;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double fp = s_f;
        int acc = 0, done = st_done;
        double eta = st_eta;
        if (a.mode == 0) {   // round start: the evaluated point is x itself; eta, done, iterations restart
            eta = a.eta0;
            done = 0;
            a.iters[b] = 0;
            a.fX[b] = fp;
            acc = 1;         // "accept": Gx <- g below (X is unchanged)
        } else {
            a.fP[b] = fp;
            if (a.checked) a.unsatP[b] = s_u;
            if (!done) {
                acc = fp <= st_fX + a.c1 * st_dot;
                eta = acc ? fmin(2.0 * eta, a.eta0) : 0.5 * eta;
                const int it = st_iters + 1;
                a.iters[b] = it;
                if (acc) a.fX[b] = fp;
                if (eta < a.eta_min || it >= a.max_inner) done = 1;
            }
        }
        a.eta[b] = eta;
        a.done[b] = done;
        const int newly = (a.checked && s_u == 0 && !st_solved) ? 1 : 0;
        if (newly) a.solved[b] = 1;
        s_acc = acc | (newly << 1);
        s_eta = eta;
        s_done = done;
    }
    __syncthreads();
    const int flags = s_acc;
    double d = 0.0;
    if (v < n) {
        const T xe = a.mode == 0 ? x0 : xp0;   // the evaluated point
        if (flags & 2) sol[v] = xe < (T)0 ? (int8_t)-1 : (int8_t)1;
        T xv = x0, gv = g0;
        if (flags & 1) {
            if (a.mode != 0) X[v] = xe;
            Gx[v] = g;
            xv = xe;
            gv = g;
        }
        // next trial point
        const T xn = s_done ? xv : clamp1(xv - (T)s_eta * gv);
        Xp[v] = xn;
        d = (double)gv * (double)(xn - xv);
    }
    // <g, x' - x>: warp sums, then the 8 warp sums in order (a fixed order)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = d;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
        a.dot[b] = t;
    }
}

// ---- accelerated projected gradient (FISTA with backtracking; "FISTA ... line search", reading #16b).
//      Per point a two-phase machine with ONE evaluation per iteration (the evaluated point is Xp, or X at a round
//      start):
//        phase 1 (Xp = clip(y - eta g_y) is a trial): accept iff f(Xp) <= f_y + <g_y, Xp - y> + |Xp - y|^2 / (2 eta)
//                (the quadratic upper bound; its right-hand side minus f_y is stored in dot[] when the trial is
//                proposed).  accept: x_prev, x <- x, Xp; t <- (1 + sqrt(1 + 4 t^2)) / 2; beta = (t_old - 1) / t;
//                eta <- min(2 eta, eta0); beta = 0: y <- Xp (f and gradient at hand), next trial; else the next
//                evaluation is y = x + beta (x - x_prev), not projected (phase 0).  reject: eta <- eta / 2, next
//                trial from the same y.
//        phase 0 (y evaluated): f_y, g_y <- f(y), grad f(y); next trial (phase 1).
//      Every evaluation counts toward max_inner; done at eta < eta_min or max_inner.  Buffers: X = x_k,
//      Xm = x_{k-1}, Y = y, Gx = g_y (the gradient at y in this mode), fX = f(x_k), fy = f(y).
struct FistaArgs {
    PgdArgs p;         // mode 0: round start (the evaluated point is X); p.dot holds <g_y, dx> + |dx|^2 / (2 eta)
    void* Xm;          // [B][n] x_{k-1}
    void* Y;           // [B][n] y
    double* fy;        // [B] f(y)
    double* t;         // [B] momentum t_k
    int32_t* phase;    // [B] 1: Xp is a trial from y; 0: Xp is the next y
};

// actions (thread 0's decision, then one pass over the point's row)
enum : int { FA_NONE = 0, FA_SETY = 1, FA_EXTRAP = 2, FA_REJECT = 3 };

// One CTA (256 threads) per point.  FUSED: the gradient / f / unsat of the evaluated point come from the TMEM path's
// point-major partials (n <= 256 = blockDim, one variable per thread); otherwise from Gp / fP / unsatP.
template <typename T, bool FUSED>
__global__ void __launch_bounds__(256) fista_step_kernel(FistaArgs fa, PmReduce<T> r) {
    pdl_wait();
    const PgdArgs& a = fa.p;
    __shared__ double s_gd[8], s_dd[8];
    __shared__ int s_act, s_flags;
    __shared__ double s_eta, s_beta, s_f;
    __shared__ int s_u;
    const int64_t b = blockIdx.x;
    const int n = a.n;
    T* X = reinterpret_cast<T*>(a.X) + b * n;
    T* Xp = reinterpret_cast<T*>(a.Xp) + b * n;
    T* Gy = reinterpret_cast<T*>(a.Gx) + b * n;
    const T* Gp = reinterpret_cast<const T*>(a.Gp) + b * n;
    T* Xm = reinterpret_cast<T*>(fa.Xm) + b * n;
    T* Y = reinterpret_cast<T*>(fa.Y) + b * n;
    int8_t* sol = a.sol + b * n;
    T gf = (T)0;
    if (FUSED) {
        if ((int)threadIdx.x < n) gf = (T)pm_grad(r, b, threadIdx.x);
        if (threadIdx.x < 32) {
            int u = 0;
            const double fb = pm_f_warp(r, b, &u);
            if (threadIdx.x == 0) {
                s_f = fb;
                s_u = u;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double fe = FUSED ? s_f : a.fP[b];
        const int ue = FUSED ? s_u : a.unsatP[b];
        double eta = a.eta[b], t = fa.t[b], beta = 0.0;
        int done = a.done[b], act = FA_NONE, acc = 0;
        if (FUSED) {
            a.fP[b] = fe;
            if (a.checked) a.unsatP[b] = ue;
        }
        if (a.mode == 0) {   // round start: the evaluated point is x itself
            eta = a.eta0;
            t = 1.0;
            done = 0;
            a.iters[b] = 0;
            a.fX[b] = fe;
            fa.fy[b] = fe;
            fa.phase[b] = 1;
            act = FA_SETY;
        } else if (!done) {
            if (fa.phase[b] == 0) {
                fa.fy[b] = fe;
                fa.phase[b] = 1;
                act = FA_SETY;
            } else if (fe <= fa.fy[b] + a.dot[b]) {
                acc = 1;
                a.fX[b] = fe;
                const double tn = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
                beta = (t - 1.0) / tn;
                t = tn;
                eta = fmin(2.0 * eta, a.eta0);
                if (beta == 0.0) {
                    fa.fy[b] = fe;
                    act = FA_SETY;
                } else {
                    fa.phase[b] = 0;
                    act = FA_EXTRAP;
                }
            } else {
                eta = 0.5 * eta;
                fa.phase[b] = 1;
                act = FA_REJECT;
            }
            const int it = a.iters[b] + 1;
            a.iters[b] = it;
            if (eta < a.eta_min || it >= a.max_inner) done = 1;
        }
        a.eta[b] = eta;
        a.done[b] = done;
        fa.t[b] = t;
        const int newly = (a.checked && ue == 0 && !a.solved[b]) ? 1 : 0;
        if (newly) a.solved[b] = 1;
        s_act = act;
        s_flags = acc | (newly << 1);
        s_eta = eta;
        s_beta = beta;
    }
    __syncthreads();
    const int act = s_act, flags = s_flags;
    const T eta = (T)s_eta, beta = (T)s_beta;
    double gd = 0.0, dd = 0.0;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        const T xe = a.mode == 0 ? X[v] : Xp[v];   // the evaluated point
        if (flags & 2) sol[v] = xe < (T)0 ? (int8_t)-1 : (int8_t)1;
        if (act == FA_NONE) continue;
        if (act == FA_EXTRAP) {
            const T xo = X[v];
            Xm[v] = xo;
            X[v] = xe;
            Xp[v] = xe + beta * (xe - xo);
            continue;
        }
        T y, gy;
        if (act == FA_SETY) {
            y = xe;
            gy = FUSED ? gf : Gp[v];
            Y[v] = y;
            Gy[v] = gy;
            if (a.mode == 0) Xm[v] = xe;
            else if (flags & 1) {   // accept with beta = 0
                Xm[v] = X[v];
                X[v] = xe;
            }
        } else {   // FA_REJECT: the next trial from the same y
            y = Y[v];
            gy = Gy[v];
        }
        const T xn = clamp1(y - eta * gy);
        Xp[v] = xn;
        const T dx = xn - y;
        gd += (double)gy * (double)dx;
        dd += (double)dx * (double)dx;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
        gd += __shfl_xor_sync(0xffffffffu, gd, o);
        dd += __shfl_xor_sync(0xffffffffu, dd, o);
    }
    if ((threadIdx.x & 31) == 0) {
        s_gd[threadIdx.x >> 5] = gd;
        s_dd[threadIdx.x >> 5] = dd;
    }
    __syncthreads();
    if (threadIdx.x == 0 && (act == FA_SETY || act == FA_REJECT)) {
        double tg = 0.0, td = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            tg += s_gd[w];
            td += s_dd[w];
        }
        a.dot[b] = tg + td / (2.0 * s_eta);
    }
}

// ---- bit-packed exact check (A9; Thm. 4, Alg. 1 line 5 P:225): the signs of 32 points of one variable
//      are one 32-bit word, so one thread checks one constraint for 32 points with one word op per literal.
// S[pt][v] bit b = 1 iff x[32 pt + b][v] < 0 (the literal "v" is True); points past B have bit 0 and are masked.
template <typename T>
__global__ void __launch_bounds__(256) signpack_kernel(const T* __restrict__ X, uint32_t* __restrict__ S, int64_t B, int32_t n) {
    const int lane = threadIdx.x & 31;
    const int64_t pt = blockIdx.y;
    const int64_t b = pt * 32 + lane;
    const bool bv = b < B;
    // warp w of block x covers 4 consecutive variables (loads all in flight; a lane's sectors are shared)
    const int64_t v0 = ((int64_t)blockIdx.x * 8 + (threadIdx.x >> 5)) * 4;
    T xv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) xv[j] = (bv && v0 + j < n) ? X[b * n + v0 + j] : (T)0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t m = __ballot_sync(0xffffffffu, xv[j] < (T)0);   // tie rule: x = 0 (either sign) is False
        if (lane == j && v0 + j < n) S[pt * n + v0 + j] = m;
    }
}

struct CheckBitsArgs {
    const uint32_t* S;        // [PT][n] sign words
    int64_t B;
    int32_t n;
    int64_t m;
    int64_t cons_per_cta;
    const int64_t* off;       // [m + 1] position-order literal offsets into words
    const uint32_t* words;    // var | neg << 31
    const int32_t* rule;      // [m][3] tmin, tmax, parity (1 odd, 2 even)
    int32_t* U;               // [m]
    int32_t* unsat;           // [B]
    int32_t skip_long;        // rows longer than kCheckLong are left to check_long_kernel
};
constexpr int kCheckLong = 128;

// Bit-sliced comparison of the per-point counts (planes p[0..13), LSB first, zero above plane P) with a constant:
// gt / eq masks (fully unrolled so the planes stay in registers).
__device__ __forceinline__ void bits_cmp(const uint32_t (&p)[13], int c, uint32_t& gt, uint32_t& eq) {
    gt = 0u;
    eq = 0xffffffffu;
    if (c >> 13) { eq = 0u; return; }   // c >= 2^13 > every count
#pragma unroll
    for (int j = 12; j >= 0; --j) {
        if ((c >> j) & 1) eq &= p[j];
        else {
            gt |= eq & p[j];
            eq &= ~p[j];
        }
    }
}

// Satisfied mask of one constraint over the 32 points of a sign tile, from its literals lo + first, lo + first +
// stride, ... (COOP: the 32 lanes of the warp take interleaved literals and the partial reductions / bit-sliced
// counts are combined across the warp, every lane ends with the result).  Literal truth masks L = S[v] ^ (negated ?
// ~0 : 0); OR / AND / parity rules reduce them with one op each, the other rules count them in bit-sliced planes
// compared with t_min / t_max.
template <bool SMEM, bool COOP>
__device__ __forceinline__ uint32_t sat_mask(const CheckBitsArgs& a, const uint32_t* S, int64_t lo, int64_t hi, int tmin, int tmax,
                                             int par, int first, int stride) {
    const int k = (int)(hi - lo);
    auto lit = [&](int64_t i) {
        const uint32_t w = __ldg(a.words + i);
        return (SMEM ? S[w & 0x7fffffffu] : __ldg(S + (w & 0x7fffffffu))) ^ (uint32_t)((int)w >> 31);
    };
    if (par == 0 && tmin == 1 && tmax >= k) {            // OR: some literal True
        uint32_t m = 0u;
        for (int64_t i = lo + first; i < hi; i += stride) m |= lit(i);
        if (COOP) m = __reduce_or_sync(0xffffffffu, m);
        return m;
    }
    if (par == 0 && tmin >= k && tmax >= k) {            // AND: every literal True
        uint32_t m = 0xffffffffu;
        for (int64_t i = lo + first; i < hi; i += stride) m &= lit(i);
        if (COOP) m = __reduce_and_sync(0xffffffffu, m);
        return tmin > k ? 0u : m;
    }
    if (par != 0 && tmin <= 0 && tmax >= k) {            // XOR / XNOR: parity of the True literals
        uint32_t x = 0u;
        for (int64_t i = lo + first; i < hi; i += stride) x ^= lit(i);
        if (COOP) x = __reduce_xor_sync(0xffffffffu, x);
        return par == 1 ? x : ~x;
    }
    // counting rules: bit-sliced planes (LSB first), k <= 4096 -> 13 planes.  The literal masks are loaded 8 at a time
    // (all in flight) before they are added: the ripple-carry adds would otherwise serialise one load latency per literal
    uint32_t p[13];
#pragma unroll
    for (int j = 0; j < 13; ++j) p[j] = 0u;
    for (int64_t i0 = lo + first; i0 < hi; i0 += 8 * (int64_t)stride) {
        uint32_t mk[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int64_t i = i0 + q * (int64_t)stride;
            mk[q] = i < hi ? lit(i) : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            uint32_t carry = mk[q];
#pragma unroll
            for (int j = 0; j < 13; ++j) {   // ripple-carry add of one bit per point
                if (carry == 0u) break;
                const uint32_t t = p[j] & carry;
                p[j] ^= carry;
                carry = t;
            }
        }
    }
    if (COOP) {   // butterfly sum of the 32 lanes' bit-sliced counts
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) {
            uint32_t carry = 0u;
#pragma unroll
            for (int j = 0; j < 13; ++j) {
                const uint32_t q = __shfl_xor_sync(0xffffffffu, p[j], d);
                const uint32_t sum = p[j] ^ q ^ carry;
                carry = (p[j] & q) | (carry & (p[j] ^ q));
                p[j] = sum;
            }
        }
    }
    uint32_t gtn, eqn, gtx, eqx;
    bits_cmp(p, tmin, gtn, eqn);
    bits_cmp(p, tmax, gtx, eqx);
    uint32_t sat = (gtn | eqn) & ~gtx;
    if (par == 1) sat &= p[0];
    if (par == 2) sat &= ~p[0];
    return sat;
}

// grid (point tiles, constraint chunks), 256 threads; SMEM: the tile's sign words staged in shared memory
// (n words), else read through the read-only path.  Thread = one constraint for 32 points (sat_mask); constraints
// longer than 128 literals are taken by the whole warp, one after the other (sat_mask<COOP>), so a long
// cardinality row does not serialise one thread.  U_c: popc of the unsat mask (one integer atomic per constraint
// with unsat points); unsat[b]: the warp transposes its 32 unsat masks with ballots, lane b keeps point b's count.
template <bool SMEM>
__global__ void __launch_bounds__(256) check_bits_kernel(CheckBitsArgs a) {
    extern __shared__ __align__(16) uint32_t sgn[];
    __shared__ int ucnt[8][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t pt = blockIdx.x, b0 = pt * 32;
    const uint32_t vm = a.B - b0 >= 32 ? 0xffffffffu : ((1u << (a.B - b0)) - 1u);
    const uint32_t* S = a.S + pt * a.n;
    if (SMEM) {
        for (int v = threadIdx.x; v < a.n; v += 256) sgn[v] = S[v];
        __syncthreads();
        S = sgn;
    }
    const int64_t c0 = (int64_t)blockIdx.y * a.cons_per_cta;
    const int64_t c1 = min(a.m, c0 + a.cons_per_cta);
    int mine = 0;   // lane b: unsat constraints of point b seen by this warp
    for (int64_t cb = c0 + warp * 32; cb < c1; cb += 256) {
        const int64_t c = cb + lane;
        uint32_t uns = 0u;
        int64_t lo = 0, hi = 0;
        int tmin = 0, tmax = 0, par = 0;
        if (c < c1) {
            lo = __ldg(a.off + c);
            hi = __ldg(a.off + c + 1);
            tmin = __ldg(a.rule + 3 * c); tmax = __ldg(a.rule + 3 * c + 1); par = __ldg(a.rule + 3 * c + 2);
        }
        const bool longc = c < c1 && hi - lo > kCheckLong && !a.skip_long;
        const bool skipped = c < c1 && hi - lo > kCheckLong && a.skip_long;
        if (c < c1 && !longc && !skipped) uns = ~sat_mask<SMEM, false>(a, S, lo, hi, tmin, tmax, par, 0, 1) & vm;
        for (uint32_t lm = __ballot_sync(0xffffffffu, longc); lm; lm &= lm - 1) {
            const int src = __ffs(lm) - 1;
            const int64_t lo_s = __shfl_sync(0xffffffffu, lo, src), hi_s = __shfl_sync(0xffffffffu, hi, src);
            const uint32_t sat = sat_mask<SMEM, true>(a, S, lo_s, hi_s, __shfl_sync(0xffffffffu, tmin, src),
                                                      __shfl_sync(0xffffffffu, tmax, src), __shfl_sync(0xffffffffu, par, src), lane, 32);
            if (lane == src) uns = ~sat & vm;
        }
        if (uns) atomicAdd(a.U + c, __popc(uns));
        // transpose: point b's count over this warp's 32 constraints = popc of the ballot of bit b
#pragma unroll 8
        for (int bb = 0; bb < 32; ++bb) {
            const int cnt = __popc(__ballot_sync(0xffffffffu, (uns >> bb) & 1u));
            if (lane == bb) mine += cnt;
        }
    }
    ucnt[warp][lane] = mine;
    __syncthreads();
    if (warp == 0 && b0 + lane < a.B) {
        int tot = 0;
        for (int w = 0; w < 8; ++w) tot += ucnt[w][lane];
        if (tot) atomicAdd(a.unsat + b0 + lane, tot);
    }
}


// Long rows (k > kCheckLong) of the round-end check, spread out: one warp per (long constraint, 32-point tile), the
// 32 lanes interleaving its literals (sat_mask COOP); U_c and the per-point counts by integer atomics (exact, order
// free).  check_bits_kernel skips these rows (a.skip_long), so a few thousand-literal rows no longer serialise on the
// one warp whose constraint range holds them.  grid (tiles, ceil(n_long / 8)), 256 threads.
template <bool SMEM>
__global__ void __launch_bounds__(256) check_long_kernel(CheckBitsArgs a, const int32_t* longs, int32_t n_long) {
    extern __shared__ __align__(16) uint32_t sgn[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t pt = blockIdx.x, b0 = pt * 32;
    const uint32_t vm = a.B - b0 >= 32 ? 0xffffffffu : ((1u << (a.B - b0)) - 1u);
    const uint32_t* S = a.S + pt * a.n;
    if (SMEM) {
        for (int v = threadIdx.x; v < a.n; v += 256) sgn[v] = S[v];
        __syncthreads();
        S = sgn;
    }
    const int j = blockIdx.y * 8 + warp;
    if (j >= n_long) return;
    const int64_t c = longs[j];
    const int64_t lo = __ldg(a.off + c), hi = __ldg(a.off + c + 1);
    const int tmin = __ldg(a.rule + 3 * c), tmax = __ldg(a.rule + 3 * c + 1), par = __ldg(a.rule + 3 * c + 2);
    const uint32_t uns = ~sat_mask<SMEM, true>(a, S, lo, hi, tmin, tmax, par, lane, 32) & vm;
    if (lane == 0 && uns) atomicAdd(a.U + c, __popc(uns));
    if ((uns >> lane) & 1u) atomicAdd(a.unsat + b0 + lane, 1);
}

// Round-end check for formulas without long rows (k <= 64): one thread per constraint over a group of TPC point
// tiles (blockIdx.y), so U_c is counted in a register (one integer atomic per constraint and tile group instead of
// one per constraint and tile) and the per-point counts of the CTA's tiles are accumulated in shared memory (ballot
// transposition per warp and tile), then added to unsat[] once per CTA.  Integer sums: exact, order-free.
template <int TPC>
__global__ void __launch_bounds__(256) check_rows_kernel(CheckBitsArgs a) {
    __shared__ int cnt[TPC * 32];
    const int lane = threadIdx.x & 31;
    const int64_t pt0 = (int64_t)blockIdx.y * TPC;
    const int64_t PT = (a.B + 31) / 32;
    const int ntile = (int)min((int64_t)TPC, PT - pt0);
    for (int i = threadIdx.x; i < TPC * 32; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool cv = c < a.m;
    int64_t lo = 0, hi = 0;
    int tmin = 0, tmax = 0, par = 0;
    if (cv) {
        lo = __ldg(a.off + c);
        hi = __ldg(a.off + c + 1);
        tmin = __ldg(a.rule + 3 * c); tmax = __ldg(a.rule + 3 * c + 1); par = __ldg(a.rule + 3 * c + 2);
    }
    int uc = 0;
    for (int t = 0; t < ntile; ++t) {
        const int64_t pt = pt0 + t, b0 = pt * 32;
        const uint32_t vm = a.B - b0 >= 32 ? 0xffffffffu : ((1u << (a.B - b0)) - 1u);
        uint32_t uns = 0u;
        if (cv) uns = ~sat_mask<false, false>(a, a.S + pt * a.n, lo, hi, tmin, tmax, par, 0, 1) & vm;
        uc += __popc(uns);
#pragma unroll 8
        for (int bb = 0; bb < 32; ++bb) {
            const int k = __popc(__ballot_sync(0xffffffffu, (uns >> bb) & 1u));
            if (lane == bb && k) atomicAdd(&cnt[t * 32 + bb], k);
        }
    }
    if (cv && uc) atomicAdd(a.U + c, uc);
    __syncthreads();
    for (int i = threadIdx.x; i < ntile * 32; i += blockDim.x)
        if (cnt[i] && pt0 * 32 + i < a.B) atomicAdd(a.unsat + pt0 * 32 + i, cnt[i]);
}

// ERWA (Prop. 3) in two grid-wide kernels: max U_c (block maxima, one integer atomicMax each: exact and
// order-free), then w = (1 - alpha) w + alpha U / max U (skipped when max U = 0).
__global__ void __launch_bounds__(256) umax_kernel(const int32_t* U, int64_t m, int32_t* umax) {
    int mx = 0;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x) mx = max(mx, U[c]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    __shared__ int wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = max(t, wm[w]);
        if (t > 0) atomicMax(umax, t);
    }
}

template <typename T>
__global__ void __launch_bounds__(256) erwa_kernel(T* w, const int32_t* U, int64_t m, double alpha, const int32_t* umax) {
    const int mx = *umax;
    if (mx == 0) return;
    const double inv = 1.0 / (double)mx;
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < m; c += (int64_t)gridDim.x * blockDim.x)
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

// Search statistics (single block) into out[0..2]: out[0] active (not converged) points; out[1] the solved key = lowest
// GLOBAL point index (point0 + b) whose solved flag is set, INT64_MAX if none; out[2] the incumbent key =
// (falsified count of sgn(x) at the last check << 32) | global point, minimised (lowest index among equal counts).
// out[1..2] are MIN-reducible across ranks as they stand (restart sharding, C1 / C4).
__global__ void __launch_bounds__(1024) stats_kernel(const int32_t* done, const int32_t* solved, const int32_t* unsat,
                                                     int64_t B, int64_t point0, int64_t* out /* [3] */) {
    __shared__ long long s_act[1024], s_sol[1024], s_best[1024];
    long long act = 0, sol = INT64_MAX, best = INT64_MAX;
    for (int64_t b = threadIdx.x; b < B; b += blockDim.x) {
        act += done[b] ? 0 : 1;
        if (solved[b] && point0 + b < sol) sol = point0 + b;
        long long key = ((long long)unsat[b] << 32) | (long long)(point0 + b);
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
        out[1] = s_sol[0];
        out[2] = s_best[0];
    }
}

// After the round-end check: a point whose rounded assignment sgn(x) falsifies nothing is solved (Thm. 4);
// record it like a solved trial (first solution kept).  One CTA per point.
template <typename T>
__global__ void __launch_bounds__(128) mark_solved_kernel(const T* X, const int32_t* unsat, int32_t* solved, int8_t* sol,
                                                          int32_t n) {
    const int64_t b = blockIdx.x;
    if (unsat[b] != 0 || solved[b]) return;
    const T* x = X + b * n;
    int8_t* a = sol + b * n;
    for (int v = threadIdx.x; v < n; v += blockDim.x) a[v] = x[v] < (T)0 ? (int8_t)-1 : (int8_t)1;
    __syncthreads();
    if (threadIdx.x == 0) solved[b] = 1;
}

// Host-buffer evaluation: flag any non-finite staged coordinate on the device instead of a host scan.
template <typename T>
__global__ void __launch_bounds__(256) nonfinite_kernel(const T* __restrict__ x, int64_t count, int32_t* flag) {
    int bad = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(x[i]);
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
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
