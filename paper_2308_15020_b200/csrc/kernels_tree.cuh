// kernels_tree.cuh -- product-tree path for long symmetric constraints (fp64): f and the exact gradient of
// FE = sum_t f(t) P(T = t) through a binary tree of Poisson-binomial polynomials, the work-efficient form of
// Prop. 2's log-depth product tree that the paper names as future work for long constraints.
//
// Per (constraint c, point b) item, with p_i = (1 - l_i) / 2 and the literal generating polynomials
// f_i(z) = (1 - p_i) + p_i z (so prod_i f_i = sum_t P(T = t) z^t, T = number of True literals):
//   bottom-up   node polynomial P_S = P_left * P_right (schoolbook convolution; leaves are blocks of 16 literals,
//               computed by the sequential Bernoulli recurrence of Alg. 5's forward pass);
//   root        FE = sum_t f(t) P_root[t] (Def. 3 / Thm. 1: the multilinear extension of the truth-by-count table)
//               = sum_s P_L[s] lambda_L[s] with the root's left child: the root product itself is never formed;
//   top-down    the linear functional L(g) = sum_t f(t) [z^t] g pushed down the tree: lambda_root = f, and for a
//               node S with children L, R: lambda_L[t] = sum_s lambda_S[t + s] P_R[s] (the functional g ->
//               L(g * prod_{j not in L} f_j) restricted to L's degree), symmetrically for R; at the root of an
//               interval rule (f = 1 - 2 [tmin <= t <= tmax]) from the children's cumulative sums in O(k);
//   leaves      for literal i in block g: dFE/dp_i = L(prod_{j != i} f_j (z - 1)) = sum_s delta_g[s] Q_i[s] with
//               delta_g[s] = lambda_g[s + 1] - lambda_g[s] and Q_i = P_g / f_i (one stable synthetic division);
//               dFE/dl_i = -dFE/dp_i / 2.
// Every quantity is a probability vector or a functional bounded by max |f| = 1 combined with convex weights, so the
// fp64 result is accurate to a few ulps times the tree depth.  Work per item ~ k^2 / 4 (bottom-up below the root) +
// k^2 / 2 (top-down below the root) fused multiply-adds, against 12 k M' (~6 k^2) FP64 instruction slots of the
// root-of-unity path.
//
// Mapping: one CTA of 512 threads per item (persistent CTAs take items from an atomic counter, longest constraints
// first; results do not depend on the assignment).  The polynomials of every tree level and two functional buffers
// live in shared memory (k <= 2048); the tree is balanced over 32-literal pairs; the levels below Lv - 4 run as 16
// warp-local subtrees.  A work unit computes R = 9 consecutive outputs of one node over a share of the inner index
// (the share's partial sums are combined with warp shuffles in a fixed order): one operand is read as a broadcast,
// the other through a register ring (one new element per step: 9 FMAs per 2 shared loads); R odd keeps the windowed
// loads of 32 lanes (stride R doubles) bank-conflict-free.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "kernels_common.cuh"
#include "kernels_eval.cuh"
#include "tree_geom.hpp"

namespace ffsat {
namespace dev {

constexpr int kTreeThreads = 512;
using tree::kTreeLeaf;
using tree::kTreeR;
using tree::kTreePF;
using tree::kTreeNR;
using tree::kTreePad;
using tree::TreeGeom;
using tree::tree_level_size;
using tree::tree_geom;
// node j of level l: first pair, pair end, degree (real literals; -1 for an empty level-1 slot), first coefficient
// (relative to a level base)
struct TreeNode {
    int a, b, deg, pos;
};
__device__ __forceinline__ TreeNode tree_node(const TreeGeom& g, const short* hs, int l, int j) {
    const int h = (1 << (g.Lv - l)) + j;
    TreeNode nd;
    nd.a = hs[h];
    nd.b = (((h + 1) & h) == 0) ? g.nu : hs[h + 1];   // the last node of a level ends at nu
    nd.deg = nd.b > nd.a ? min(g.k, 2 * kTreeLeaf * nd.b) - 2 * kTreeLeaf * nd.a : -1;
    nd.pos = (j + 1) * kTreePad + 2 * kTreeLeaf * nd.a + j;
    return nd;
}

// acc[r] += sum_{s = sa}^{sb - 1} A[s] W[t0 + r - s] (CONV) or A[s] W[t0 + r + s] (CORR), r = 0..R-1.  A is read as
// a (mostly) broadcast operand, W through a register ring of R + PF elements (one new element per step); the loads
// may run up to R + PF elements past the window's range on either side (the zero guards).
template <bool CONV>
__device__ __forceinline__ void tree_unit(const double* A, const double* W, int t0, int sa, int sb, double (&acc)[kTreeR]) {
    constexpr int R = kTreeR, PF = kTreePF, NR = kTreeNR;
    double ring[NR];
    // window element e' (relative): CONV index t0 - sa + e' with e' = r - u; CORR index t0 + sa + e' with e' = r + u
    const double* wp = W + (CONV ? t0 - sa : t0 + sa);
#pragma unroll
    for (int e = 0; e < R; ++e) ring[e] = wp[e];
#pragma unroll
    for (int e = 1; e < PF; ++e) {
        if (CONV) ring[NR - e] = wp[-e];
        else ring[R + e - 1] = wp[R + e - 1];
    }
    const int n = sb - sa;
    const double* ap = A + sa;
    int u0 = 0;
    for (; u0 + NR <= n; u0 += NR) {
        double av[NR];
#pragma unroll
        for (int u = 0; u < NR; ++u) av[u] = ap[u0 + u];
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            if (CONV) ring[(NR - ((u + PF) % NR)) % NR] = wp[-(u0 + u) - PF];
            else ring[(u + R + PF - 1) % NR] = wp[u0 + u + R + PF - 1];
#pragma unroll
            for (int r = 0; r < R; ++r) acc[r] = fma(av[u], ring[CONV ? (r - u + NR * 2) % NR : (r + u) % NR], acc[r]);
        }
    }
    const int rem = n - u0;
    if (rem > 0) {
        double av[NR];
#pragma unroll
        for (int u = 0; u < NR; ++u) av[u] = u < rem ? ap[u0 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < NR; ++u) {
            if (u < rem) {
                if (CONV) ring[(NR - ((u + PF) % NR)) % NR] = wp[-(u0 + u) - PF];
                else ring[(u + R + PF - 1) % NR] = wp[u0 + u + R + PF - 1];
#pragma unroll
                for (int r = 0; r < R; ++r) acc[r] = fma(av[u], ring[CONV ? (r - u + NR * 2) % NR : (r + u) % NR], acc[r]);
            }
        }
    }
}

// inner-index shares per unit: the count that keeps nt threads busiest
__device__ __forceinline__ int tree_shares(int units, int nt) {
    int best = 1;
    double be = 0.0;
    for (int P = 1; P <= 8; P *= 2) {
        const int items = units * P;
        const int rounds = (items + nt - 1) / nt;
        const double eff = (double)items / ((double)rounds * nt);
        if (eff > be + 0.02) {
            be = eff;
            best = P;
        }
    }
    return best;
}

// sum of the P partials of a unit held by P consecutive lanes (butterfly: every lane ends with the same, fixed-order sum)
__device__ __forceinline__ void tree_combine(double (&acc)[kTreeR], int P) {
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
        if (o >= P) break;
#pragma unroll
        for (int r = 0; r < kTreeR; ++r) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    }
}

// The two leaf-block polynomials of a level-1 node by the whole warp: half-warp hw (lanes 16 hw .. 16 hw + 15) forms
// block `a + hw`'s 17 coefficients (lane t of the half holds q[t], its lane 15 also q[16]) with one shuffle per literal
// (the same recurrence, q_t <- (1 - p_i) q_t + p_i q_{t-1}); an absent block (present = false) is the polynomial 1.
// Written to out[hw * 17 + t].
__device__ __forceinline__ void tree_leaf_pair(const double* p, bool present, double* out) {
    const int lane = threadIdx.x & 31, t = lane & 15, hw = lane >> 4;
    double q = t == 0 ? 1.0 : 0.0, q16 = 0.0;
#pragma unroll
    for (int i = 0; i < kTreeLeaf; ++i) {
        const double pi = present ? p[i] : 0.0;
        const double qm = __shfl_up_sync(0xffffffffu, q, 1, 16);
        const double q15 = q;
        q = fma(pi, t == 0 ? 0.0 : qm, (1.0 - pi) * q);
        q16 = fma(pi, q15, (1.0 - pi) * q16);
    }
    out[hw * (kTreeLeaf + 1) + t] = q;
    if (t == 15) out[hw * (kTreeLeaf + 1) + 16] = q16;
}

__device__ __forceinline__ double tree_f(int t, const SymSigDev& sg) { return rule_sat(t, sg.tmin, sg.tmax, sg.parity) ? -1.0 : 1.0; }

// fixed-order CTA sums (warp butterflies, then the warps in order)
__device__ __forceinline__ double tree_block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < kTreeThreads / 32; ++w) t += red[w];
    return t;
}

// Inclusive prefix sums out[i] = in[0] + ... + in[i], i < len, by the CTA in a fixed order (each thread a contiguous
// segment, then the segment totals scanned by warp shuffles and the warps in order): deterministic.
__device__ __forceinline__ void tree_block_scan(const double* in, double* out, int len, double* s_tot) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int seg = (len + kTreeThreads - 1) / kTreeThreads;
    const int i0 = tid * seg, i1 = min(len, i0 + seg);
    double run = 0.0;
    for (int i = i0; i < i1; ++i) run += in[i];
    double inc = run;   // warp-inclusive scan of the segment totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    __syncthreads();
    if (lane == 31) s_tot[warp] = inc;
    __syncthreads();
    double off = inc - run;
    for (int w = 0; w < warp; ++w) off += s_tot[w];
    for (int i = i0; i < i1; ++i) {
        off += in[i];
        out[i] = off;
    }
    __syncthreads();
}

// Bottom-up level l >= 2: the polynomials of nodes [j0, j1) from their children, by threads ti of nt (nt a multiple of
// 32; whole warps take part: the share sums use shuffles).  Units of kTreeR outputs x P inner-index shares.
__device__ __forceinline__ void tree_up_level(const TreeGeom& g, const short* hs, double* sm, int l, int j0, int j1, int ti, int nt) {
    const int nl = j1 - j0;
    const int maxdeg = 2 * kTreeLeaf * ((g.nu + (1 << (g.Lv - l)) - 1) >> (g.Lv - l));
    const int nbF = (maxdeg + 1 + kTreeR - 1) / kTreeR;
    const int units = nl * nbF;
    const int P = tree_shares(units, nt);
    const int items = (units * P + 31) / 32 * 32;
    for (int w = ti; w < items; w += nt) {
        const int q = w / P, h = w - q * P;
        const int jr = q / nbF, t0 = (q - jr * nbF) * kTreeR, j = j0 + jr;
        TreeNode nd{0, 0, -1, 0};
        if (jr < nl) nd = tree_node(g, hs, l, j);
        const bool ok = t0 <= nd.deg;
        int sa = 0, sb = 0;
        const double *A = sm, *W = sm;
        if (ok) {
            const TreeNode cA = tree_node(g, hs, l - 1, 2 * j);
            TreeNode cB = tree_node(g, hs, l - 1, 2 * j + 1);
            if (cB.deg < 0) cB.deg = 0;   // an empty right child (level 1 only): the polynomial 1
            A = sm + g.off[l - 1] + cA.pos;
            W = cB.b > cB.a ? sm + g.off[l - 1] + cB.pos : sm + g.one + kTreePad;
            const int lo_s = max(0, t0 - cB.deg), hi_s = min(cA.deg, t0 + kTreeR - 1);
            int per = (hi_s - lo_s + P) / P;
            per += P > 1 ? 1 - (per & 1) : 0;   // odd: the P shares' broadcast reads fall in distinct banks
            sa = min(hi_s + 1, lo_s + h * per);
            sb = min(hi_s + 1, sa + per);
        }
        double acc[kTreeR];
#pragma unroll
        for (int r = 0; r < kTreeR; ++r) acc[r] = 0.0;
        if (sa < sb) tree_unit<true>(A, W, t0, sa, sb, acc);
        tree_combine(acc, P);
        if (ok && h == 0) {
            double* dst = sm + g.off[l] + nd.pos;
#pragma unroll
            for (int r = 0; r < kTreeR; ++r)
                if (t0 + r <= nd.deg) dst[t0 + r] = acc[r];
        }
    }
}

// Top-down from level l >= 2: the functionals of the children of nodes [j0, j1) (parents in buffer cur, children into
// nxt): lambda_L = corr(lambda_S, P_R), lambda_R = corr(lambda_S, P_L).  Reads past a parent's end only feed outputs
// past the child's degree, which are not stored (the buffers hold finite values: zeroed at kernel start).
__device__ __forceinline__ void tree_down_level(const TreeGeom& g, const short* hs, double* sm, int l, int j0, int j1, int cur, int nxt,
                                                int ti, int nt) {
    const int nl = j1 - j0;
    const int maxdeg = 2 * kTreeLeaf * ((g.nu + (2 << (g.Lv - l)) - 1) >> (g.Lv - l + 1));   // of a child
    const int nbF = (maxdeg + 1 + kTreeR - 1) / kTreeR;
    const int units = nl * 2 * nbF;
    const int P = tree_shares(units, nt);
    const int items = (units * P + 31) / 32 * 32;
    for (int w = ti; w < items; w += nt) {
        const int q = w / P, h = w - q * P;
        const int jr = q / (2 * nbF), rq = q - jr * 2 * nbF, side = rq / nbF, t0 = (rq - side * nbF) * kTreeR;
        const int j = j0 + jr, child = 2 * j + side;
        TreeNode cd{0, 0, -1, 0};
        if (jr < nl) cd = tree_node(g, hs, l - 1, child);
        const bool ok = t0 <= cd.deg;
        int sa = 0, sb = 0;
        const double *A = sm, *W = sm;
        if (ok) {
            const TreeNode sib = tree_node(g, hs, l - 1, 2 * j + 1 - side);
            const TreeNode par = tree_node(g, hs, l, j);
            A = sib.deg >= 0 ? sm + g.off[l - 1] + sib.pos : sm + g.one + kTreePad;   // empty sibling: 1
            W = sm + cur + par.pos;
            const int hi_s = max(sib.deg, 0);
            int per = (hi_s + P) / P;
            per += P > 1 ? 1 - (per & 1) : 0;
            sa = min(hi_s + 1, h * per);
            sb = min(hi_s + 1, sa + per);
        }
        double acc[kTreeR];
#pragma unroll
        for (int r = 0; r < kTreeR; ++r) acc[r] = 0.0;
        if (sa < sb) tree_unit<false>(A, W, t0, sa, sb, acc);
        tree_combine(acc, P);
        if (ok && h == 0) {
            double* dst = sm + nxt + cd.pos;
#pragma unroll
            for (int r = 0; r < kTreeR; ++r)
                if (t0 + r <= cd.deg) dst[t0 + r] = acc[r];
        }
    }
}

// Level-1 node j (one warp): the two leaf-block polynomials (kept at g.leaf for the leaf stage) and their product,
// the node's polynomial (p is zero past k, so a missing or partial second block is exact).
__device__ __forceinline__ void tree_leaf_up(const TreeGeom& g, const short* hs, double* sm, const double* p, int j) {
    const int lane = threadIdx.x & 31;
    const TreeNode nd = tree_node(g, hs, 1, j);
    if (nd.deg < 0) return;   // an empty slot (warp-uniform)
    double* tw = sm + g.leaf + j * 2 * (kTreeLeaf + 1);
    tree_leaf_pair(p + 2 * kTreeLeaf * nd.a + kTreeLeaf * (lane >> 4), true, tw);
    __syncwarp();
    double* dst = sm + g.off[1] + nd.pos;
    for (int t = lane; t <= nd.deg; t += 32) {
        double c = 0.0;
        for (int u = max(0, t - kTreeLeaf); u <= min(kTreeLeaf, t); ++u) c = fma(tw[u], tw[kTreeLeaf + 1 + t - u], c);
        dst[t] = c;
    }
    __syncwarp();
}

// Leaf stage of level-1 node j (one warp, lane = literal 32 a + lane): the two block functionals from the node's
// functional (at lamb), then per literal dFE/dp_i = sum_s (lambda[s + 1] - lambda[s]) Q_i[s], where the block's
// leave-one-out polynomial Q_i = P_block / f_i comes from ONE synthetic division by the linear factor f_i = (1 - p_i)
// + p_i z, run in the stable direction: ascending when p_i <= 1/2 (each step multiplies the carried error by
// p_i / (1 - p_i) <= 1), descending from the top otherwise ((1 - p_i) / p_i <= 1); terms into Tb.
__device__ __forceinline__ void tree_leaf_down(const TreeGeom& g, const short* hs, double* sm, const double* lamb, const double* p,
                                               int j, double* tw, const SymArgs<double>& a, int64_t lo, int64_t b, double wc) {
    const int lane = threadIdx.x & 31;
    const TreeNode nd = tree_node(g, hs, 1, j);
    if (nd.deg < 0) return;
    const double* lam1 = lamb + nd.pos;
    const double* PL = sm + g.leaf + j * 2 * (kTreeLeaf + 1);   // P_L, P_R (from the bottom-up pass)
    // lambda_L[t] = sum_s lam1[t + s] P_R[s], lambda_R[t] = sum_s lam1[t + s] P_L[s], t = 0..16
    if (lane <= kTreeLeaf) {
        double vl = 0.0, vr = 0.0;
        for (int u = 0; u <= kTreeLeaf; ++u) {
            vl = fma(lam1[lane + u], PL[kTreeLeaf + 1 + u], vl);
            vr = fma(lam1[lane + u], PL[u], vr);
        }
        tw[lane] = vl;
        tw[kTreeLeaf + 1 + lane] = vr;
    }
    __syncwarp();
    const int blk = lane >> 4;
    const int i = 2 * kTreeLeaf * nd.a + lane;
    if (i < g.k) {
        const double* P = PL + blk * (kTreeLeaf + 1);
        const double pi = p[i];
        double q[kTreeLeaf];
        if (pi <= 0.5) {
            const double r = 1.0 / (1.0 - pi);
            double prev = 0.0;
#pragma unroll
            for (int t = 0; t < kTreeLeaf; ++t) {
                q[t] = fma(-pi, prev, P[t]) * r;
                prev = q[t];
            }
        } else {
            const double r = 1.0 / pi, qi = 1.0 - pi;
            double nxt = 0.0;
#pragma unroll
            for (int t = kTreeLeaf; t >= 1; --t) {
                q[t - 1] = fma(-qi, nxt, P[t]) * r;
                nxt = q[t - 1];
            }
        }
        const double* lb = tw + blk * (kTreeLeaf + 1);
        double dp = 0.0;
#pragma unroll
        for (int u = 0; u < kTreeLeaf; ++u) dp = fma(lb[u + 1] - lb[u], q[u], dp);
        const uint32_t w = __ldg(a.words + lo + i);
        const double v = wc * (-0.5 * dp);   // dFE/dl_i = -dFE/dp_i / 2
        a.Tb[(a.tb_fast + lo + i) * a.B + b] = (int)w < 0 ? -v : v;
    }
    __syncwarp();
}

__global__ void __launch_bounds__(kTreeThreads, 1) sym_tree_kernel(SymArgs<double> a, int64_t s_begin, int64_t n_items, int32_t* counter,
                                                                    int32_t smem_doubles) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double s_red[kTreeThreads / 32];
    __shared__ short s_hs[512];    // first pair of each tree node, heap order (root 1, children 2h, 2h + 1)
    __shared__ int s_item;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NW = kTreeThreads / 32;
    // every buffer starts finite (the functional buffers are never re-zeroed: see tree_down_level)
    for (int i = tid; i < smem_doubles; i += kTreeThreads) sm[i] = 0.0;
    for (;;) {
        if (tid == 0) s_item = atomicAdd(counter, 1);
        __syncthreads();
        const int64_t item = s_item;
        if (item >= n_items) break;
        const int64_t s = s_begin + item / a.B, b = item - (item / a.B) * a.B;   // the class is sorted by k, longest first
        const SymSigDev sg = a.sigs[a.sig_of[s]];
        const TreeGeom g = tree_geom(sg.k);
        const int k = g.k;
        const int64_t lo = a.off[s];
        // the polynomial levels (guards and unused tails must read as 0), the constant 1; then p_i = (1 - l_i) / 2
        for (int i = g.kp + tid; i < g.lamX; i += kTreeThreads) sm[i] = 0.0;
        for (int i = g.one + tid; i < g.scr; i += kTreeThreads) sm[i] = 0.0;
        double* p = sm;
        int tc = 0;
        for (int i = tid; i < g.kp; i += kTreeThreads) {
            double pi = 0.0;
            if (i < k) {
                const uint32_t w = __ldg(a.words + lo + i);
                const double xv = a.x[b * a.sb + (int64_t)(w & 0x7fffffffu) * a.sv];
                const double l = (int)w < 0 ? -xv : xv;
                pi = 0.5 - 0.5 * l;
                tc += (int)((xv < 0.0) != ((int)w < 0));   // the literal is True (sgn rounding, x = 0 -> False)
            }
            p[i] = pi;
        }
        // balanced node ranges, level by level from the root (one warp)
        if (warp == 0) {
            if (lane == 0) s_hs[1] = 0;
            for (int l = g.Lv; l >= 2; --l) {
                __syncwarp();
                const int h0 = 1 << (g.Lv - l);
                for (int h = h0 + lane; h < 2 * h0; h += 32) {
                    const int na = s_hs[h], nbb = (((h + 1) & h) == 0) ? g.nu : s_hs[h + 1];
                    s_hs[2 * h] = (short)na;
                    s_hs[2 * h + 1] = (short)(na + (nbb - na + 1) / 2);
                }
            }
        }
        __syncthreads();
        if (tid == 0) sm[g.one + kTreePad] = 1.0;   // (ordered after the zeroing above; read after the next barrier)
        // warp-local subtrees: rooted at level lw = Lv - 4 (16 of them, one per warp), or at level 1 for small trees
        const int lw = max(1, g.Lv - 4), nsub = 1 << (g.Lv - lw), w1 = 1 << (lw - 1);
        double* tw = sm + g.scr + warp * 2 * (kTreeLeaf + 1);
        // ---- bottom-up: levels 1..lw per warp, then lw+1..Lv by the CTA
        for (int r = warp; r < nsub; r += NW) {
            for (int j = r * w1; j < (r + 1) * w1; ++j) tree_leaf_up(g, s_hs, sm, p, j);
            for (int l = 2; l <= lw; ++l) {
                tree_up_level(g, s_hs, sm, l, r << (lw - l), (r + 1) << (lw - l), lane, 32);
                __syncwarp();
            }
        }
        // (the root's own product is never formed: FE comes from its left child below)
        for (int l = lw + 1; l < g.Lv; ++l) {
            __syncthreads();
            tree_up_level(g, s_hs, sm, l, 0, 1 << (g.Lv - l), tid, kTreeThreads);
        }
        __syncthreads();
        // ---- root functional lambda = f
        double* lam = sm + g.lamX + kTreePad;
        for (int t = tid; t <= k; t += kTreeThreads) lam[t] = tree_f(t, sg);
        __syncthreads();
        // ---- top-down: levels Lv..lw+1 by the CTA, then lw..2 and the leaves per warp
        int cur = g.lamX, nxt = g.lamY;
        double fe = 0.0;
        for (int l = g.Lv; l > lw; --l) {
            if (l == g.Lv && sg.parity == 0) {
                // root of an interval rule (satisfied iff tmin <= t <= tmax: f = 1 - 2 [tmin <= t <= tmax]): the root's
                // correlations in O(k) from the children's cumulative sums, lambda_L[s] = sum_u f(s + u) P_R[u] =
                // T_R - 2 (C_R(tmax - s) - C_R(tmin - s - 1)) (C_R(i) = sum_{u <= i} P_R[u], 0 for i < 0), likewise R
                const TreeNode cl = tree_node(g, s_hs, g.Lv - 1, 0), cr = tree_node(g, s_hs, g.Lv - 1, 1);
                double* CL = sm + cur;                     // lambda_root = f is not needed on this path: scratch
                double* CR = sm + cur + cl.deg + 1;
                tree_block_scan(sm + g.off[g.Lv - 1] + cl.pos, CL, cl.deg + 1, s_red);
                tree_block_scan(sm + g.off[g.Lv - 1] + cr.pos, CR, cr.deg + 1, s_red);
                const double TL = CL[cl.deg], TR = CR[cr.deg];
                auto cdf = [](const double* C, int d, int i) { return i < 0 ? 0.0 : C[min(i, d)]; };
                for (int t = tid; t <= cl.deg; t += kTreeThreads)
                    sm[nxt + cl.pos + t] = TR - 2.0 * (cdf(CR, cr.deg, sg.tmax - t) - cdf(CR, cr.deg, sg.tmin - t - 1));
                for (int t = tid; t <= cr.deg; t += kTreeThreads)
                    sm[nxt + cr.pos + t] = TL - 2.0 * (cdf(CL, cl.deg, sg.tmax - t) - cdf(CL, cl.deg, sg.tmin - t - 1));
            } else {
                tree_down_level(g, s_hs, sm, l, 0, 1 << (g.Lv - l), cur, nxt, tid, kTreeThreads);
            }
            __syncthreads();
            if (l == g.Lv) {   // FE = L(P_L P_R) = sum_s P_L[s] lambda_L[s] (lambda_L = corr(f, P_R), just formed)
                const TreeNode cl = tree_node(g, s_hs, g.Lv - 1, 0);
                const double* pl = sm + g.off[g.Lv - 1] + cl.pos;
                const double* ll = sm + nxt + cl.pos;
                double v = 0.0;
                for (int t = tid; t <= cl.deg; t += kTreeThreads) v = fma(pl[t], ll[t], v);
                fe = tree_block_sum(v, s_red);
            }
            const int tsw = cur;
            cur = nxt;
            nxt = tsw;
        }
        const double wc = a.w_sym[s];
        for (int r = warp; r < nsub; r += NW) {
            int c = cur, x = nxt;
            for (int l = lw; l >= 2; --l) {
                tree_down_level(g, s_hs, sm, l, r << (lw - l), (r + 1) << (lw - l), c, x, lane, 32);
                __syncwarp();
                const int tsw = c;
                c = x;
                x = tsw;
            }
            for (int j = r * w1; j < (r + 1) * w1; ++j) tree_leaf_down(g, s_hs, sm, sm + c, p, j, tw, a, lo, b, wc);
        }
        // unsat count (integer, exact), f
        int tcs = tc;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) tcs += __shfl_xor_sync(0xffffffffu, tcs, o);
        __syncthreads();
        if (lane == 0) reinterpret_cast<int*>(s_red)[warp] = tcs;
        __syncthreads();
        if (tid == 0) {
            int t = 0;
            for (int w = 0; w < NW; ++w) t += reinterpret_cast<int*>(s_red)[w];
            a.fsym[s * a.B + b] = wc * fe;
            a.usym[s * a.B + b] = rule_sat(t, sg.tmin, sg.tmax, sg.parity) ? 0 : 1;
        }
        __syncthreads();
    }
}

}  // namespace dev
}  // namespace ffsat
