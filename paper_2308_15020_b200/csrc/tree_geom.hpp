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
constexpr size_t kTreeSmemMax = 226 * 1024;   // dynamic shared memory of one tree CTA (227 KB minus the static part)

// Shared-memory layout of one item (doubles), a function of k only (host: tree_smem_doubles mirrors it).
struct TreeGeom {
    int k, kp, Lv;               // kp = k rounded up to 32; levels 1..Lv (level l node = 16 << l literals)
    int off[12];                 // level l polynomial region (l = 1..Lv); off[0] = the p array
    int lamX, lamY, lamSize;     // the two functional buffers (each sized for the largest level)
    int one;                     // the constant polynomial 1 surrounded by zeros
    int total;
};

FFSAT_HD inline int tree_nodes(int k, int l) { const int D = kTreeLeaf << l; return (k + D - 1) / D; }
FFSAT_HD inline int tree_level_size(int k, int l, int Lv) {
    const int D = kTreeLeaf << l;
    return l == Lv ? 2 * kTreePad + k + 1 : kTreePad + tree_nodes(k, l) * (D + 1 + kTreePad);
}
FFSAT_HD inline TreeGeom tree_geom(int k) {
    TreeGeom g{};
    g.k = k;
    g.kp = (k + 31) / 32 * 32;
    int Lv = 1;
    while (tree_nodes(k, Lv) > 1) ++Lv;
    g.Lv = Lv;
    int o = g.kp;
    g.off[0] = 0;
    for (int l = 1; l <= Lv; ++l) {
        g.off[l] = o;
        o += tree_level_size(k, l, Lv);
    }
    // the functional buffers hold any level's functionals, and the per-warp scratch of the leaf phase (16 x 68)
    g.lamSize = 16 * 4 * (kTreeLeaf + 1);
    for (int l = 1; l <= Lv; ++l) g.lamSize = g.lamSize > tree_level_size(k, l, Lv) ? g.lamSize : tree_level_size(k, l, Lv);
    g.lamX = o;
    g.lamY = o + g.lamSize;
    g.one = g.lamY + g.lamSize;
    g.total = g.one + 2 * kTreePad + 1;
    return g;
}

// FP64 instructions of one item on the tree path (the algorithmic count of the roofline): one DFMA per
// multiply-add of the level convolutions (bottom-up, levels 2..Lv) and correlations (top-down, levels Lv..2) over the
// real degrees, plus the level-1 / leaf stage.
inline int64_t tree_fp64_work(int k) {
    const TreeGeom g = tree_geom(k);
    auto deg = [&](int l, int j) { const int D = kTreeLeaf << l; const int d = k - j * D; return d < D ? d : D; };
    int64_t w = 0;
    const int n1 = tree_nodes(k, 1);
    // per level-1 node: the two leaf recurrences twice (bottom-up and leaf stage; 136 updates of 2 slots each), the
    // 17 x 17 product, the two 17 x 17 leaf functionals; per literal: its leave-one-out recurrence and 16-term dot
    w += (int64_t)n1 * (4 * 2 * 136 + 17 * 17 + 2 * 17 * 17);
    w += (int64_t)k * (2 * 136 + 2 * 16);
    for (int l = 2; l <= g.Lv; ++l)
        for (int j = 0; j < tree_nodes(k, l); ++j) {
            const int dA = deg(l - 1, 2 * j), dB = deg(l - 1, 2 * j + 1);
            if (dB <= 0) continue;
            w += (int64_t)(dA + 1) * (dB + 1) * 3;   // bottom-up product + the two top-down correlations
        }
    return w;
}

}  // namespace tree
}  // namespace ffsat
