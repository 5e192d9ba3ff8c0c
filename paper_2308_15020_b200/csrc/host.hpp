// host.hpp -- host-side formula layer of libffsat (steps A1-A3 of DESIGN.md):
// parse + validate (A1), classify / bucket / CSR layouts (A2), per-signature fp64
// coefficient tables (A3).  Plain C++17, no CUDA.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ffsat.h"

namespace ffsat {

struct Error : std::runtime_error {
    ffsat_status code;
    Error(ffsat_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct Formula {
    int32_t n = 0;
    std::vector<uint8_t> kind;
    std::vector<int32_t> bound;
    std::vector<double> weight;
    std::vector<int64_t> offsets{0};
    std::vector<int32_t> lits;
    int64_t m() const { return (int64_t)kind.size(); }
};

Formula parse_text(const std::string& text);           // throws Error (FFSAT_ERR_PARSE/RANGE/DUPVAR/BOUND)
Formula from_arrays(const ffsat_formula& f);           // copies
void validate(const Formula& F);                       // throws Error

// Satisfaction of a constraint as an interval of the True-count t plus a parity rule:
// satisfied iff tmin <= t <= tmax and (parity == 0 || (parity == 1 && t odd) || (parity == 2 && t even)).
struct SatRule { int32_t tmin, tmax, parity; };
SatRule sat_rule(int kind, int k, int bound);

// Fast-path variants (PAPER.md footnote P:964 and App. B):
// FE = g0 + gA * A + gB * Bp + gX * X with A = prod (1+l)/2, Bp = prod (1-l)/2, X = prod l.
enum Variant : int32_t { V_OR = 0, V_AND, V_NAE, V_XOR, V_XNOR, V_TRUE, V_NOR, V_NAND, V_COUNT };
struct FastForm { int32_t variant; double g0, gA, gB, gX; };
bool fast_form(int kind, int k, int bound, FastForm* out);

struct FastBucket {
    int32_t variant, k, kp;        // kp = k rounded up to a multiple of 4 (16-byte literal rows)
    bool own = false;              // global path, k <= kOwnKMax: gradient by owner-computes (no T slots)
    int64_t pos_begin, pos_end;    // constraint positions (layout order)
    int64_t word_off;              // first padded literal word of the bucket
    int64_t slot_off;              // first (unpadded) literal slot of the bucket
    double g0, gA, gB, gX;
    SatRule rule;
};

inline int fast_nch(const FastBucket& b) { return (b.gA != 0) + (b.gB != 0) + (b.gX != 0); }   // product channels
constexpr int kFastKMax = 64;       // fast product paths handle k <= 64; longer constraints use roots

struct SymSig {                     // a (k, sat rule) signature with its root table
    int32_t k, tmin, tmax, parity, Mp;  // Mp = floor((k+1)/2) roots m = 1..Mp
    int64_t coef_off;               // 8 doubles per root: alpha(re,im) beta(re,im) G(re,im) H(re,im)
    double g0;
};

struct SymClass {                   // launch class: G threads per (constraint, point), C literals per thread
                                    // (G = 0: one thread per item, C = the literal bound KMAX)
    int32_t G, C, R;                // R roots per pass
    int64_t begin, end;             // sym constraint indices
    int32_t max_mp;                 // largest M' in the class (root-table size staged in shared memory)
    int32_t S = 1;                  // root splits: each item's M' roots are shared by S CTAs (balance; G > 0 only)
    int64_t lit_begin = 0, lit_end = 0;   // the class's literals in the sym word array
};
constexpr int kRootChunk = 256;     // target roots per CTA of the root path (SymClass::S = ceil(max M' / kRootChunk)); c3: 64 -> 1.77 ms, 128 -> 1.69, 256 -> 1.68, unsplit 1.85

struct WorkUnit {                   // a run of fast constraints of one bucket, contiguous positions
    int32_t bucket;                 // tiled path: a var-disjoint class (no variable occurs twice in it),
    int32_t count;                  // so the warps of a CTA can add its terms into the shared gradient
    int64_t pos_begin;              // tile concurrently and deterministically
};

constexpr int kTreeClass = -1;      // SymClass::G of the product-tree path
bool tree_path(int k, int precision);   // fp64 long symmetric constraints whose tree fits in shared memory
int sym_group(int k);               // threads per (constraint, point) on the root path
int sym_chunk(int k);               // literals per thread on the root path (G * C >= k)
int sym_roots(int k);               // roots per pass on the root path

struct Layout {
    int32_t n = 0, path = 0, precision = 32, max_k = 0;
    bool wide = false;                  // tiled path with 64 points per CTA (fp32, uniform single-channel k <= 16)
    bool tmem = false;                  // ... with the gradient tile in tensor memory (n <= 256; else shared memory)
    int32_t wide_red = 0;               // the bit reduction (1 OR, 2 AND, 3 XOR) shared by every fast bucket, or 0
    int64_t m = 0, L = 0;
    std::vector<int64_t> order;     // position -> original constraint index (fast first, then sym)
    std::vector<int64_t> pos_of;    // original constraint index -> position
    std::vector<double> w_pos;      // static weight by position
    // fast
    int64_t n_fast = 0, n_fast_lits = 0, n_fast_words = 0;
    std::vector<FastBucket> fbuckets;
    std::vector<uint32_t> fast_words;   // var | neg << 31 (padded rows)
    // sym
    int64_t n_sym = 0, n_sym_lits = 0, sym_root_lits = 0;
    std::vector<SymSig> sigs;
    std::vector<double> coef;
    std::vector<int32_t> sym_sig;       // per sym constraint
    std::vector<int64_t> sym_off;       // [n_sym + 1] literal offsets into sym_words
    std::vector<uint32_t> sym_words;    // var | neg << 31
    std::vector<int32_t> sym_rule;      // 3 ints per sym constraint (tmin, tmax, parity)
    std::vector<SymClass> sym_classes;
    bool sym_lane = false;              // some root-path class runs thread-per-item on x^T (needs the transpose)
    int64_t n_tree_cons = 0;            // sym constraints on the product-tree path (kernels_tree.cuh; SymClass G = kTreeClass)
    int64_t tree_work = 0;              // its FP64 instructions per point (tree::tree_fp64_work summed)
    // T-buffer slots (global path: non-owner fast slots then sym slots; tiled path: sym slots only)
    int64_t tb_fast = 0, tb_slots = 0;
    // owner-computes (global path, fast buckets with k <= kOwnKMax): per variable its occurrences in those
    // constraints, ascending position, as self-contained 16-byte records {position, the other literals' words (in
    // literal order, padded with the first), bucket << 8 | literal index << 1 | own literal negated}
    bool own_sliced = false;        // every fast constraint is owner-computed and nothing else reads x^T: x^T is laid out in
                                    // 16-point slices [B/16][n][16] so one slice (n x 64 B) stays L2-resident per pass
    bool own = false;
    int32_t own_uni = -1;               // the single owner bucket when there is exactly one (owner_grp_kernel), else -1
    int64_t n_own_lits = 0;
    std::vector<int64_t> own_off;       // [n + 1]
    std::vector<uint32_t> own_rec;      // 4 per occurrence
    // the single-bucket case (owner_grp_kernel) instead: per block of 8 G variable slots (G = 32 / own_lanes), 8 groups
    // of G (the variables of each 8-block window sorted by occurrence counts and dealt in that order to the window's
    // blocks; grp_var: slot -> variable, -1 past n); per group {record offset lo, hi,
    // rows A, rows B}; its records interleaved [row][G slots], rows A = the occurrences at literal index 0 (ascending
    // position), rows B = the others (ascending position), each padded to the group's longest list with pad records
    // {0, 0, 0, 2}.  Record {position, the other literals' words (literal order), bit 0 own negated | bit 1 pad}
    int32_t own_wpb = 1;                // owner_grp_kernel: warps (groups) per CTA (the records' blocks of 8 groups
                                        // are split over 8 / own_wpb CTAs; FFSAT_OWN_WPB),
    int32_t own_ppt = 4;                // ... points per thread,
    int32_t own_lanes = 8;              // ... threads per variable (x^T slices of own_lanes * own_ppt points; groups of
                                        // 32 / own_lanes variables, blocks of 8 groups, windows of 8 blocks); 1 (one
                                        // point, a warp over 32 variables) for single-point plans (batch_ref <= 4)
    std::vector<uint32_t> grp_desc;     // 4 per group
    std::vector<int32_t> grp_var;       // [32 * ceil(n / 32)]
    std::vector<uint32_t> grp_rec;      // 4 per record (incl. pads)
    std::vector<int64_t> occ_off;       // [n + 1]
    std::vector<int64_t> occ_slot;      // ascending slot ids per variable
    // work units of the fast kernels (tiled: var-disjoint classes; global: runs of <= 512 literals)
    std::vector<WorkUnit> units;
    std::vector<int64_t> unit_rows;     // literals per unit (chunk balancing)
    std::vector<uint32_t> tiled_words;  // tiled path: (var * kTilePitch) | neg << 31 (padded rows)
};

constexpr int kOwnSlice = 8;       // points per x^T slice of the sliced owner-computes path (one slice's x^T stays in L2)
constexpr int kOwnSliceMax = 32;   // the widest slice (owner_grp_kernel, 8 lanes x 4 points per thread)
constexpr int kOwnLanes = 8;       // owner_grp_kernel: threads per variable (default; FFSAT_OWN_LANES)
constexpr int kOwnKMax = 3;         // global path, FFSAT_OWN=1: constraints this short take the owner-computes gradient
constexpr int kTilePitch = 66;      // smem row pitch of the tiled kernel: x half-row (32 points + pad) | gradient half-row
constexpr int kClassCap = 16;
constexpr int kWidePitch = 132;     // wide tiled kernel row: x (64 points + 2 pad) | gradient (64 + 2)       // constraints per var-disjoint class (2 per warp of an 8-warp CTA)

// Build everything; path: 0 auto, 1 tiled, 2 global; precision 0 auto / 32 / 64.
Layout build_layout(const Formula& F, int path, int precision, int64_t batch_ref = 1024);
// Tiled-path admission: the max n whose x and gradient tiles fit shared memory for the dtype.
int tiled_max_n(int precision);
size_t tiled_smem_bytes(int n, int precision);
int wide_max_n();                   // largest n for the wide (64-point) fp32 tiled kernel
size_t wide_smem_bytes(int n);
size_t tmem_smem_bytes(int n);      // the TMEM kernel's dynamic shared memory: x tile [n][64] fp32 (>= the f / unsat exchange)
uint32_t tmem_cols(int n);          // TMEM columns it allocates: the power of two >= 2 n (>= 32)
constexpr int kTmemMaxN = 256;
// Greedy partition of one bucket's constraints into var-disjoint classes of at most `cap` members
// (first fit over the most recent `window` open classes).  Returns class id per constraint.
std::vector<int32_t> disjoint_classes(const std::vector<std::vector<int32_t>>& vars, int32_t n, int cap, int window);

}  // namespace ffsat
