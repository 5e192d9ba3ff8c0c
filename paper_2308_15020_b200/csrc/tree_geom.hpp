// tree_geom.hpp -- shared-memory geometry of the product-tree kernel (kernels_tree.cuh), shared with the host layout
// (host.cpp decides which constraints fit the tree path and counts its work).
#pragma once
#include <cstddef>
#include <cstdint>
#ifdef __CUDACC__
#define FFSAT_HD __host__ __device__
#else
#define FFSAT_HD
#endif

namespace ffsat {
namespace tree {

constexpr int kTreeLeaf = 16;    // literals per leaf block
constexpr int kTreeR = 9;        // outputs per work unit
constexpr int kTreePF = 3;       // window elements loaded ahead
constexpr int kTreeNR = kTreeR + kTreePF;
constexpr int kTreePad = 16;     // zero guard before / after every node (>= kTreeR + kTreePF)
constexpr size_t kTreeSmemMax = 224 * 1024;   // dynamic shared memory of one tree CTA (227 KB minus the static part, 2.2 KB)

// Shared-memory layout of one item (doubles), a function of k only.  Level-1 nodes are pairs of 16-literal leaf blocks
// (32 literals, the last one partial); above them the tree is BALANCED over the nu = ceil(k / 32) pairs: a node
// covering pairs [a, b) splits at a + ceil((b - a) / 2), so siblings differ by at most one pair (uniform work per
// level).  Level l (1..Lv, Lv = 1 + ceil(log2 nu)) has 2^(Lv - l) node slots; every node above level 1 holds >= 1
// pair, a level-1 slot holds 1 or 0 (an empty right child).  Node j of level l is stored compactly: its deg + 1
// coefficients at off[l] + (j + 1) kTreePad + 32 start_j + j, zero guards between.
struct TreeGeom {
    int k, kp, nu, Lv;           // kp = 32 nu (the p array, zero past k)
    int off[12];                 // level l polynomial region (l = 1..Lv)
    int lamX, lamY, lamSize;     // the two functional buffers (each sized for the largest level)
    int one;                     // the constant polynomial 1 surrounded by zeros
    int scr;                     // per-warp scratch
    int leaf;                    // leaf-block polynomials (kept from the bottom-up pass for the leaf stage)
    int total;
};

FFSAT_HD inline int tree_level_size(int k, int l, int Lv) {
    const int nl = 1 << (Lv - l);
    return (nl + 1) * kTreePad + k + nl;
}
FFSAT_HD inline TreeGeom tree_geom(int k) {
    TreeGeom g{};
    g.k = k;
    g.nu = (k + 2 * kTreeLeaf - 1) / (2 * kTreeLeaf);
    g.kp = 2 * kTreeLeaf * g.nu;
    int Lv = 1;
    while ((1 << (Lv - 1)) < g.nu) ++Lv;
    g.Lv = Lv;
    int o = g.kp;
    for (int l = 1; l <= Lv; ++l) {
        g.off[l] = o;
        o += tree_level_size(k, l, Lv);
    }
    // the functional buffers hold any level's functionals
    g.lamSize = 0;
    for (int l = 1; l <= Lv; ++l) g.lamSize = g.lamSize > tree_level_size(k, l, Lv) ? g.lamSize : tree_level_size(k, l, Lv);
    g.lamX = o;
    g.lamY = o + g.lamSize;
    g.one = g.lamY + g.lamSize;
    g.scr = g.one + 2 * kTreePad + 1;          // per-warp scratch of the leaf stage: 16 x 2 x 17
    g.leaf = g.scr + 16 * 2 * (kTreeLeaf + 1);  // the two leaf-block polynomials of every level-1 slot (34 each)
    g.total = g.leaf + (1 << (Lv - 1)) * 2 * (kTreeLeaf + 1);
    return g;
}

// FP64 instructions of one item on the tree path (the algorithmic count of the roofline): one DFMA per
// multiply-add of the level convolutions (bottom-up, levels 2..Lv) and correlations (top-down, levels Lv..2) over the
// real degrees, plus the level-1 / leaf stage.
inline int64_t tree_fp64_work(int k, int parity) {
    const TreeGeom g = tree_geom(k);
    // node pair ranges, heap order (root 1, children 2h, 2h + 1), as the kernel builds them
    int64_t start[1 << 10], endb[1 << 10];
    start[1] = 0;
    endb[1] = g.nu;
    for (int h = 1; h < (1 << (g.Lv - 1)); ++h) {
        const int64_t a = start[h], b = endb[h];
        start[2 * h] = a;
        endb[2 * h] = a + (b - a + 1) / 2;
        start[2 * h + 1] = endb[2 * h];
        endb[2 * h + 1] = b;
    }
    auto deg = [&](int h) { const int64_t e = endb[h] * 2 * kTreeLeaf < k ? endb[h] * 2 * kTreeLeaf : k; const int64_t d = e - start[h] * 2 * kTreeLeaf; return d > 0 ? d : 0; };
    int64_t w = 0;
    // per level-1 node: the two leaf recurrences (136 updates of 2 slots each), the 17 x 17 product, the two 17 x 17
    // leaf functionals; per literal: its leave-one-out polynomial by one 16-step division (2 slots a step) and the
    // 16-term dot (2 slots a term)
    w += (int64_t)g.nu * (2 * 2 * 136 + 17 * 17 + 2 * 17 * 17);
    w += (int64_t)k * (2 * 16 + 2 * 16);
    for (int h = 1; h < (1 << (g.Lv - 1)); ++h) {   // nodes of levels 2..Lv
        const int64_t dA = deg(2 * h), dB = deg(2 * h + 1);
        // bottom-up product + the two top-down correlations; at the root no product (FE comes from its left child's
        // functional: dA + 1 FMAs) and, for an interval rule (parity 0), the correlations from cumulative sums (~4 k)
        if (dB > 0) {
            if (h != 1) w += (dA + 1) * (dB + 1) * 3;
            else w += (parity == 0 ? 4 * (dA + dB + 2) : (dA + 1) * (dB + 1) * 2) + dA + 1;
        }
    }
    return w;
}

}  // namespace tree
}  // namespace ffsat
