// host.cpp -- host formula layer of libffsat: A1 parse/validate, A2 bucketing and CSR layouts,
// A3 coefficient tables.  See host.hpp and DESIGN.md.
#include "host.hpp"
#include "tree_geom.hpp"

#include <algorithm>
#include <cstdlib>
#include <array>
#include <cerrno>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>
#include <sstream>

namespace ffsat {

// ------------------------------------------------------------------------------- A1: parse

static bool parse_int(const std::string& s, long long* v) {
    if (s.empty()) return false;
    char* end = nullptr;
    errno = 0;
    long long r = std::strtoll(s.c_str(), &end, 10);
    if (errno || *end) return false;
    *v = r;
    return true;
}

Formula parse_text(const std::string& text) {
    Formula F;
    bool have_header = false, weighted = false, cnf = false;
    std::istringstream in(text);
    std::string line;
    long long lineno = 0;
    std::vector<int32_t> stamp;
    auto fail = [&](ffsat_status c, const std::string& msg) {
        throw Error(c, "line " + std::to_string(lineno) + ": " + msg);
    };
    while (std::getline(in, line)) {
        ++lineno;
        std::istringstream ls(line);
        std::vector<std::string> tok;
        for (std::string t; ls >> t;) tok.push_back(t);
        if (tok.empty() || tok[0] == "c" || tok[0][0] == '%') continue;
        if (tok[0] == "p") {
            long long n, m;
            if (have_header) fail(FFSAT_ERR_PARSE, "second header");
            if (tok.size() != 4 || (tok[1] != "cnf" && tok[1] != "hnf" && tok[1] != "whnf") ||
                !parse_int(tok[2], &n) || !parse_int(tok[3], &m) || n < 0 || n > INT32_MAX || m < 0)
                fail(FFSAT_ERR_PARSE, "bad header (expected 'p cnf|hnf|whnf <n> <m>')");
            F.n = (int32_t)n;
            cnf = tok[1] == "cnf";
            weighted = tok[1] == "whnf";
            have_header = true;
            stamp.assign((size_t)n + 1, -1);
            continue;
        }
        if (!have_header) fail(FFSAT_ERR_PARSE, "constraint before header");
        size_t i = 0;
        double w = 1.0;
        if (weighted) {
            char* end = nullptr;
            w = std::strtod(tok[0].c_str(), &end);
            if (*end) fail(FFSAT_ERR_PARSE, "bad weight '" + tok[0] + "'");
            if (!std::isfinite(w)) fail(FFSAT_ERR_NONFINITE, "non-finite weight");
            ++i;
        }
        int kind = FFSAT_OR;
        long long bound = 0;
        if (!cnf) {
            if (i >= tok.size()) fail(FFSAT_ERR_PARSE, "missing constraint tag");
            const std::string& tag = tok[i++];
            if (tag == "o") kind = FFSAT_OR;
            else if (tag == "x") kind = FFSAT_XOR;
            else if (tag == "xn") kind = FFSAT_XNOR;
            else if (tag == "n") kind = FFSAT_NAE;
            else if (tag == "d" || tag == "a") {
                kind = tag == "d" ? FFSAT_CARD_GE : FFSAT_CARD_LE;
                if (i >= tok.size() || !parse_int(tok[i], &bound)) fail(FFSAT_ERR_PARSE, "bad cardinality bound");
                ++i;
            } else fail(FFSAT_ERR_PARSE, "unknown constraint tag '" + tag + "'");
        }
        if (tok.back() != "0") fail(FFSAT_ERR_PARSE, "constraint not terminated by 0");
        int32_t cidx = (int32_t)F.kind.size();
        int64_t k = 0;
        for (; i + 1 < tok.size(); ++i) {
            long long v;
            if (!parse_int(tok[i], &v) || v == 0) fail(FFSAT_ERR_PARSE, "bad literal '" + tok[i] + "'");
            long long a = v < 0 ? -v : v;
            if (a > F.n) fail(FFSAT_ERR_RANGE, "literal " + tok[i] + " out of range");
            if (stamp[(size_t)a] == cidx) fail(FFSAT_ERR_DUPVAR, "duplicate variable " + std::to_string(a));
            stamp[(size_t)a] = cidx;
            F.lits.push_back((int32_t)v);
            ++k;
        }
        if (k == 0) fail(FFSAT_ERR_PARSE, "empty constraint");
        if ((kind == FFSAT_CARD_GE || kind == FFSAT_CARD_LE) && (bound < 0 || bound > k))
            fail(FFSAT_ERR_BOUND, "cardinality bound out of range");
        F.kind.push_back((uint8_t)kind);
        F.bound.push_back((int32_t)bound);
        F.weight.push_back(w);
        F.offsets.push_back((int64_t)F.lits.size());
    }
    if (!have_header) throw Error(FFSAT_ERR_PARSE, "line " + std::to_string(lineno) + ": missing header");
    return F;
}

Formula from_arrays(const ffsat_formula& f) {
    if (f.n_vars < 0 || f.n_cons < 0) throw Error(FFSAT_ERR_ARG, "negative sizes");
    if (f.n_cons > 0 && (!f.kind || !f.offsets || !f.lits)) throw Error(FFSAT_ERR_ARG, "null formula arrays");
    Formula F;
    F.n = f.n_vars;
    int64_t m = f.n_cons;
    if (m == 0) return F;
    if (f.offsets[0] != 0) throw Error(FFSAT_ERR_ARG, "offsets[0] must be 0");
    for (int64_t c = 0; c < m; ++c)
        if (f.offsets[c + 1] < f.offsets[c]) throw Error(FFSAT_ERR_ARG, "offsets must be non-decreasing");
    int64_t L = f.offsets[m];
    F.kind.assign(f.kind, f.kind + m);
    F.bound.assign((size_t)m, 0);
    if (f.bound) F.bound.assign(f.bound, f.bound + m);
    F.weight.assign((size_t)m, 1.0);
    if (f.weight) F.weight.assign(f.weight, f.weight + m);
    F.offsets.assign(f.offsets, f.offsets + m + 1);
    F.lits.assign(f.lits, f.lits + L);
    return F;
}

void validate(const Formula& F) {
    std::vector<int64_t> stamp((size_t)F.n + 1, -1);
    for (int64_t c = 0; c < F.m(); ++c) {
        std::string where = "constraint " + std::to_string(c);
        if (F.kind[c] > FFSAT_NAE) throw Error(FFSAT_ERR_ARG, where + ": unknown kind");
        int64_t k = F.offsets[c + 1] - F.offsets[c];
        if (k <= 0) throw Error(FFSAT_ERR_ARG, where + ": empty constraint");
        if (!std::isfinite(F.weight[c])) throw Error(FFSAT_ERR_NONFINITE, where + ": non-finite weight");
        if ((F.kind[c] == FFSAT_CARD_GE || F.kind[c] == FFSAT_CARD_LE) && (F.bound[c] < 0 || F.bound[c] > k))
            throw Error(FFSAT_ERR_BOUND, where + ": cardinality bound out of range");
        for (int64_t i = F.offsets[c]; i < F.offsets[c + 1]; ++i) {
            int64_t v = F.lits[i];
            int64_t a = v < 0 ? -v : v;
            if (v == 0 || a > F.n) throw Error(FFSAT_ERR_RANGE, where + ": literal out of range");
            if (stamp[(size_t)a] == c) throw Error(FFSAT_ERR_DUPVAR, where + ": duplicate variable " + std::to_string(a));
            stamp[(size_t)a] = c;
        }
    }
}

// ------------------------------------------------------------------------------- classification

SatRule sat_rule(int kind, int k, int bound) {
    switch (kind) {
    case FFSAT_OR: return {1, k, 0};
    case FFSAT_XOR: return {0, k, 1};
    case FFSAT_XNOR: return {0, k, 2};
    case FFSAT_CARD_GE: return {bound, k, 0};
    case FFSAT_CARD_LE: return {0, bound, 0};
    case FFSAT_NAE: return {1, k - 1, 0};
    }
    return {1, 0, 0};
}

bool fast_form(int kind, int k, int bound, FastForm* o) {
    *o = FastForm{V_OR, 0, 0, 0, 0};
    if (k > kFastKMax) return false;  // long constraints of any kind take the root-product path
    if (kind == FFSAT_XOR) { *o = {V_XOR, 0, 0, 0, 1}; return true; }
    if (kind == FFSAT_XNOR) { *o = {V_XNOR, 0, 0, 0, -1}; return true; }
    if (kind == FFSAT_NAE) { *o = {V_NAE, -1, 2, 2, 0}; return true; }
    if (kind == FFSAT_OR || (kind == FFSAT_CARD_GE && bound == 1)) { *o = {V_OR, -1, 2, 0, 0}; return true; }
    if ((kind == FFSAT_CARD_GE && bound == 0) || (kind == FFSAT_CARD_LE && bound == k)) { *o = {V_TRUE, -1, 0, 0, 0}; return true; }
    if (kind == FFSAT_CARD_GE && bound == k) { *o = {V_AND, 1, 0, -2, 0}; return true; }
    if (kind == FFSAT_CARD_LE && bound == 0) { *o = {V_NOR, 1, -2, 0, 0}; return true; }
    if (kind == FFSAT_CARD_LE && bound == k - 1) { *o = {V_NAND, -1, 0, 2, 0}; return true; }
    return false;
}

// ------------------------------------------------------------------------------- A3: coefficients

// g_m = 1/(k+1) sum_t f(t) w^{-tm}, w = exp(-2 pi i/(k+1)) (P:151 sign, #1); f(t) = -1 on the
// satisfying interval, +1 elsewhere.  Root-product factors alpha_m + beta_m l with alpha = (1+w^m)/2,
// beta = (1-w^m)/2 (probability basis); G_m = 2 g_m except the Nyquist root.
static void sym_coefficients(int k, SatRule r, std::vector<double>& coef, double* g0_out, int* Mp_out) {
    const int K1 = k + 1;
    std::vector<long double> cs(K1), sn(K1);
    const long double two_pi = 6.283185307179586476925286766559005768L;
    for (int j = 0; j < K1; ++j) {
        long double a = two_pi * (long double)j / (long double)K1;
        cs[j] = cosl(a);
        sn[j] = sinl(a);
    }
    std::vector<int> f(K1);
    long double s0 = 0;
    for (int t = 0; t <= k; ++t) {
        bool sat = t >= r.tmin && t <= r.tmax && (r.parity == 0 || (r.parity == 1) == ((t & 1) == 1));
        f[t] = sat ? -1 : 1;
        s0 += f[t];
    }
    *g0_out = (double)(s0 / K1);
    const int Mp = K1 / 2;
    *Mp_out = Mp;
    for (int m = 1; m <= Mp; ++m) {
        long double re = 0, im = 0;  // sum_t f(t) e^{+2 pi i t m/(k+1)} = sum_t f(t) w^{-tm}
        for (int t = 0; t <= k; ++t) {
            int j = (int)(((long long)t * m) % K1);
            re += f[t] * cs[j];
            im += f[t] * sn[j];
        }
        long double gre = re / K1, gim = im / K1;
        long double mult = (2 * m == K1) ? 1.0L : 2.0L;
        long double Gre = mult * gre, Gim = mult * gim;
        // w^m = exp(-2 pi i m / K1) = cos - i sin
        int jm = m % K1;
        long double wr = cs[jm], wi = -sn[jm];
        long double ar = (1 + wr) / 2, ai = wi / 2;
        long double br = (1 - wr) / 2, bi = -wi / 2;
        long double Hr = Gre * br - Gim * bi, Hi = Gre * bi + Gim * br;
        double row[8] = {(double)ar, (double)ai, (double)br, (double)bi, (double)Gre, (double)Gim, (double)Hr, (double)Hi};
        coef.insert(coef.end(), row, row + 8);
    }
}

// ------------------------------------------------------------------------------- tiled sizing

size_t tiled_smem_bytes(int n, int precision) {
    size_t es = precision == 64 ? 8 : 4;
    // x tile and gradient tile [n][kTilePitch]; at least 3 KB (the kernel's final f / unsat exchange)
    return std::max<size_t>(es * (size_t)kTilePitch * (size_t)n, 3072);
}

size_t wide_smem_bytes(int n) { return std::max<size_t>(4 * (size_t)kWidePitch * (size_t)n, 6144); }  // >= the final f / unsat exchange (8 x 64 x 12 B)
size_t tmem_smem_bytes(int n) { return std::max<size_t>(2 * 260 * (size_t)n, 12288); }   // 2 sum tiles [n][65] (the x tile is the first); >= 16 x 64 x 12 B
uint32_t tmem_cols(int n) {
    uint32_t c = 32;
    while (c < 2u * (uint32_t)n) c <<= 1;
    return c;
}

int wide_max_n() {
    const size_t budget = 227 * 1024 - 4608;
    int n = 0;
    while (wide_smem_bytes(n + 1) <= budget) ++n;
    return n;
}

int tiled_max_n(int precision) {
    const size_t budget = 227 * 1024 - 4608;   // minus the kernel's static stage buffers
    int n = 0;
    while (tiled_smem_bytes(n + 1, precision) <= budget) ++n;
    return n;
}

std::vector<int32_t> disjoint_classes(const std::vector<std::vector<int32_t>>& vars, int32_t n, int cap, int window) {
    const size_t words = ((size_t)n + 63) / 64;
    std::vector<std::vector<uint64_t>> mask;   // per class
    std::vector<int32_t> fill;
    std::vector<int32_t> open;                 // most recent open classes, oldest first
    std::vector<int32_t> cls(vars.size());
    for (size_t c = 0; c < vars.size(); ++c) {
        int32_t got = -1;
        for (size_t j = 0; j < open.size() && got < 0; ++j) {
            const std::vector<uint64_t>& mk = mask[(size_t)open[j]];
            bool ok = true;
            for (int32_t v : vars[c])
                if (mk[(size_t)v >> 6] >> (v & 63) & 1ull) { ok = false; break; }
            if (ok) {
                got = open[j];
                if (fill[(size_t)got] + 1 >= cap) open.erase(open.begin() + (long)j);
            }
        }
        if (got < 0) {
            got = (int32_t)mask.size();
            mask.emplace_back(words, 0ull);
            fill.push_back(0);
            if (cap > 1) open.push_back(got);
            if ((int)open.size() > window) open.erase(open.begin());
        }
        for (int32_t v : vars[c]) mask[(size_t)got][(size_t)v >> 6] |= 1ull << (v & 63);
        fill[(size_t)got] += 1;
        cls[c] = got;
    }
    return cls;
}

// ------------------------------------------------------------------------------- A2: layout

// Root path launch geometry.  k <= 32: one thread per item (sym_lane_kernel); k <= 128: one warp, four per lane.
// Longer: the smallest of a short ladder of (NW warps, C literals per thread) capacities 32 NW C that holds
// k -- padding slots cost full root-sweep work, so the ladder keeps them under ~25% (typically ~10%), while
// keeping the number of distinct launch classes small (each class is one launch on its own side stream).
static void sym_geom(int k, int* nw_out, int* c_out) {
    // k <= 32: thread per (constraint, point) item (sym_lane_kernel), "nw" 0, c = the register bound KMAX
    if (k <= 32) { *nw_out = 0; *c_out = k <= 8 ? 8 : k <= 16 ? 16 : 32; return; }
    if (k <= 128) { *nw_out = 1; *c_out = 4; return; }
    static const int ladder[][2] = {{1, 8}, {1, 16}, {2, 12}, {2, 16}, {4, 10}, {3, 16}, {4, 14}, {4, 16}, {6, 16}, {8, 16}};
    for (const auto& g : ladder)
        if (32 * g[0] * g[1] >= k) { *nw_out = g[0]; *c_out = g[1]; return; }
    throw Error(FFSAT_ERR_ARG, "root-path constraint too long for one thread group (k > 4096)");
}
int sym_chunk(int k) { int nw, c; sym_geom(k, &nw, &c); return c; }
// Product-tree path (kernels_tree.cuh): fp64 symmetric constraints of at least FFSAT_TREE_KMIN literals (default 256;
// FFSAT_TREE=0 keeps every constraint on the root-of-unity path) whose tree fits in one CTA's shared memory.
bool tree_path(int k, int precision) {
    if (precision != 64) return false;
    const char* e0 = std::getenv("FFSAT_TREE");
    const char* e1 = std::getenv("FFSAT_TREE_KMIN");
    const bool on = !(e0 && std::atoi(e0) == 0);
    const int kmin = e1 ? std::max(33, std::atoi(e1)) : 256;
    return on && k >= kmin && (size_t)tree::tree_geom(k).total * 8 <= tree::kTreeSmemMax;
}
// roots per pass: 1 with the factors kept in registers (measured faster than recomputing them for a
// higher occupancy or than two roots per pass: profiles/r01_bench_c3_*.json)
int sym_roots(int) { return 1; }
int sym_group(int k) { int nw, c; sym_geom(k, &nw, &c); return 32 * nw; }

Layout build_layout(const Formula& F, int path, int precision, int64_t batch_ref) {
    Layout Lo;
    Lo.n = F.n;
    Lo.m = F.m();
    Lo.L = F.lits.size();
    const int64_t m = F.m();
    std::vector<FastForm> ff((size_t)m);
    std::vector<char> is_fast((size_t)m, 0);
    bool need64 = false;
    for (int64_t c = 0; c < m; ++c) {
        int k = (int)(F.offsets[c + 1] - F.offsets[c]);
        Lo.max_k = std::max(Lo.max_k, k);
        is_fast[c] = fast_form(F.kind[c], k, F.bound[c], &ff[c]);
        if (!is_fast[c]) {
            if (k > 4096) throw Error(FFSAT_ERR_ARG, "constraint " + std::to_string(c) + ": cardinality length > 4096 unsupported");
            if (k > 64) need64 = true;
        }
    }
    if (precision == 0) precision = need64 ? 64 : 32;
    if (precision != 32 && precision != 64) throw Error(FFSAT_ERR_ARG, "precision must be 0, 32 or 64");
    Lo.precision = precision;

    // fast buckets keyed by (k, variant), sym grouped by (G class, k, rule)
    std::vector<int64_t> fast_ids, sym_ids;
    for (int64_t c = 0; c < m; ++c) (is_fast[c] ? fast_ids : sym_ids).push_back(c);
    auto klen = [&](int64_t c) { return (int)(F.offsets[c + 1] - F.offsets[c]); };
    std::stable_sort(fast_ids.begin(), fast_ids.end(), [&](int64_t a, int64_t b) {
        int ka = klen(a), kb = klen(b);
        if (ka != kb) return ka < kb;
        return ff[a].variant < ff[b].variant;
    });
    // launch geometry of a sym constraint: the product-tree class (G = kTreeClass, sorted last) or a root-path class
    auto sgeom = [&](int k, int* G, int* C) {
        if (tree_path(k, precision)) { *G = kTreeClass; *C = 1 << 20; return; }
        *G = sym_group(k);
        *C = sym_chunk(k);
    };
    std::stable_sort(sym_ids.begin(), sym_ids.end(), [&](int64_t a, int64_t b) {
        int ga, gb, ca, cb;
        sgeom(klen(a), &ga, &ca);
        sgeom(klen(b), &gb, &cb);
        if (ca != cb) return ca < cb;
        if (ga != gb) return ga > gb;   // largest groups first (longest work first within a launch)
        return klen(a) > klen(b);
    });

    // ---- path: tiled (x and gradient tiles in shared memory) when n fits, else global
    const bool allow_wide = path != 3;   // 3 = tiled path with the 32-point kernel only (tests)
    const bool allow_tmem = path != 4;   // 4 = tiled path without the TMEM kernel (the shared-memory 64-point kernel)
    if (path == 3 || path == 4) path = 1;
    if (path == 0) path = (!fast_ids.empty() && F.n <= tiled_max_n(precision)) ? 1 : 2;
    if (path == 1 && F.n > tiled_max_n(precision)) throw Error(FFSAT_ERR_ARG, "tiled path needs n <= " + std::to_string(tiled_max_n(precision)));
    if (path != 1 && path != 2) throw Error(FFSAT_ERR_ARG, "path must be 0 .. 4");
    Lo.path = path;

    // ---- tiled path: within each (k, variant) run, group constraints into var-disjoint classes and make
    //      each class a contiguous position range (the kernel's warps add a class's terms concurrently)
    std::vector<int32_t> fast_class;   // class id (global over runs) per fast position
    if (path == 1) {
        std::vector<int64_t> reordered;
        reordered.reserve(fast_ids.size());
        size_t r0 = 0;
        int32_t class_base = 0;
        while (r0 < fast_ids.size()) {
            size_t r1 = r0;
            const int k = klen(fast_ids[r0]);
            while (r1 < fast_ids.size() && klen(fast_ids[r1]) == k && ff[fast_ids[r1]].variant == ff[fast_ids[r0]].variant) ++r1;
            std::vector<std::vector<int32_t>> vars(r1 - r0);
            for (size_t j = r0; j < r1; ++j)
                for (int64_t i = F.offsets[fast_ids[j]]; i < F.offsets[fast_ids[j] + 1]; ++i)
                    vars[j - r0].push_back((F.lits[i] > 0 ? F.lits[i] : -F.lits[i]) - 1);
            const int cap = (int)std::max<int64_t>(1, std::min<int64_t>(kClassCap, (int64_t)(0.6 * F.n) / std::max(1, k)));
            std::vector<int32_t> cls = disjoint_classes(vars, F.n, cap, 64);
            int32_t ncls = 0;
            for (int32_t c : cls) ncls = std::max(ncls, c + 1);
            std::vector<std::vector<int64_t>> members((size_t)ncls);
            for (size_t j = r0; j < r1; ++j) members[(size_t)cls[j - r0]].push_back(fast_ids[j]);
            for (int32_t q = 0; q < ncls; ++q)
                for (int64_t c : members[(size_t)q]) {
                    reordered.push_back(c);
                    fast_class.push_back(class_base + q);
                }
            class_base += ncls;
            r0 = r1;
        }
        fast_ids.swap(reordered);
    }
    Lo.order = fast_ids;
    Lo.order.insert(Lo.order.end(), sym_ids.begin(), sym_ids.end());
    Lo.pos_of.assign((size_t)m, 0);
    for (int64_t p = 0; p < m; ++p) Lo.pos_of[Lo.order[p]] = p;
    Lo.w_pos.resize((size_t)m);
    for (int64_t p = 0; p < m; ++p) Lo.w_pos[p] = F.weight[Lo.order[p]];

    // ---- fast layout
    Lo.n_fast = (int64_t)fast_ids.size();
    for (int64_t p = 0; p < Lo.n_fast; ++p) {
        int64_t c = fast_ids[p];
        int k = klen(c);
        if (Lo.fbuckets.empty() || Lo.fbuckets.back().k != k || Lo.fbuckets.back().variant != ff[c].variant) {
            FastBucket b{};
            b.variant = ff[c].variant;
            b.k = k;
            b.kp = (k + 3) / 4 * 4;
            b.pos_begin = p;
            b.word_off = Lo.n_fast_words;
            b.slot_off = Lo.n_fast_lits;
            b.g0 = ff[c].g0; b.gA = ff[c].gA; b.gB = ff[c].gB; b.gX = ff[c].gX;
            b.rule = sat_rule(F.kind[c], k, F.bound[c]);
            Lo.fbuckets.push_back(b);
        }
        FastBucket& b = Lo.fbuckets.back();
        b.pos_end = p + 1;
        for (int i = 0; i < b.kp; ++i) {
            uint32_t w = 0;
            if (i < k) {
                int32_t lit = F.lits[F.offsets[c] + i];
                w = (uint32_t)((lit > 0 ? lit : -lit) - 1) | (lit < 0 ? 0x80000000u : 0u);
            }
            Lo.fast_words.push_back(w);
        }
        Lo.n_fast_words += b.kp;
        Lo.n_fast_lits += k;
    }

    // ---- sym layout
    Lo.n_sym = (int64_t)sym_ids.size();
    Lo.sym_off.push_back(0);
    std::vector<std::array<int, 4>> sig_keys;
    for (int64_t s = 0; s < Lo.n_sym; ++s) {
        int64_t c = sym_ids[s];
        int k = klen(c);
        SatRule r = sat_rule(F.kind[c], k, F.bound[c]);
        std::array<int, 4> key{k, r.tmin, r.tmax, r.parity};
        int sig = -1;
        for (size_t q = 0; q < sig_keys.size(); ++q)
            if (sig_keys[q] == key) { sig = (int)q; break; }
        if (sig < 0) {
            SymSig S{};
            S.k = k; S.tmin = r.tmin; S.tmax = r.tmax; S.parity = r.parity;
            S.coef_off = (int64_t)Lo.coef.size() / 8;
            sym_coefficients(k, r, Lo.coef, &S.g0, &S.Mp);
            sig = (int)Lo.sigs.size();
            Lo.sigs.push_back(S);
            sig_keys.push_back(key);
        }
        Lo.sym_sig.push_back(sig);
        Lo.sym_rule.push_back(r.tmin); Lo.sym_rule.push_back(r.tmax); Lo.sym_rule.push_back(r.parity);
        for (int i = 0; i < k; ++i) {
            int32_t lit = F.lits[F.offsets[c] + i];
            Lo.sym_words.push_back((uint32_t)((lit > 0 ? lit : -lit) - 1) | (lit < 0 ? 0x80000000u : 0u));
        }
        Lo.n_sym_lits += k;
        if (!tree_path(k, precision)) Lo.sym_root_lits += (int64_t)k * ((k + 1) / 2);   // root-of-unity path only
        Lo.sym_off.push_back(Lo.n_sym_lits);
        int G, C;
        sgeom(k, &G, &C);
        const int R = G == kTreeClass ? 0 : sym_roots(k);
        if (G == kTreeClass) {
            Lo.n_tree_cons += 1;
            Lo.tree_work += tree::tree_fp64_work(k, r.parity);
        }
        if (Lo.sym_classes.empty() || Lo.sym_classes.back().G != G || Lo.sym_classes.back().C != C)
            Lo.sym_classes.push_back({G, C, R, s, s + 1, 0});
        else Lo.sym_classes.back().end = s + 1;
        Lo.sym_classes.back().max_mp = std::max(Lo.sym_classes.back().max_mp, (k + 1) / 2);
        if (G == 0) Lo.sym_lane = true;
    }
    // roots per CTA of the root path (FFSAT_ROOT_CHUNK overrides kRootChunk: a tuning knob)
    int root_chunk = kRootChunk;
    if (const char* e = std::getenv("FFSAT_ROOT_CHUNK")) root_chunk = std::max(1, std::atoi(e));
    for (SymClass& cl : Lo.sym_classes) {
        cl.lit_begin = Lo.sym_off[(size_t)cl.begin];
        cl.lit_end = Lo.sym_off[(size_t)cl.end];
        cl.S = cl.G <= 0 ? 1 : std::max(1, std::min(32, (cl.max_mp + root_chunk - 1) / root_chunk));
    }

    // ---- owner-computes buckets (global path): no T slots; the other fast buckets' slots are renumbered densely.
    // ON by default when the global path's fast constraints form ONE bucket of short constraints (k <= 3: uniform
    // random 3-SAT, c5) and no root-path class reads x^T: x^T in 32-point slices and the grouped-record kernel
    // (owner_grp_kernel: c5 evaluation 1.34 -> 0.92 ms, 2.4 GB of DRAM traffic instead of 4.7 GB).
    // FFSAT_OWN=1 forces it for every global-path bucket with k <= 3 (owner_grad_kernel for mixed buckets: measured
    // slower than the T-buffer path), FFSAT_OWN=0 turns it off.
    int own_kmax = 0;
    {
        bool short_only = path == 2 && !Lo.fbuckets.empty();
        for (const FastBucket& b : Lo.fbuckets) short_only = short_only && b.k <= kOwnKMax;
        if (const char* e = std::getenv("FFSAT_OWN")) own_kmax = (path == 2 && std::atoi(e) != 0) ? kOwnKMax : 0;
        else if (short_only && Lo.fbuckets.size() == 1 && !Lo.sym_lane) own_kmax = kOwnKMax;
        Lo.own_sliced = own_kmax > 0 && short_only && !Lo.sym_lane;
    }
    {
        int64_t ts = 0;
        for (FastBucket& b : Lo.fbuckets) {
            b.own = b.k <= own_kmax;
            b.slot_off = b.own ? 0 : ts;
            if (!b.own) ts += (b.pos_end - b.pos_begin) * b.k;
            else Lo.n_own_lits += (b.pos_end - b.pos_begin) * b.k;
        }
        if (path == 2) Lo.tb_fast = ts;
        Lo.own = Lo.n_own_lits > 0;
        int nown = 0;
        for (size_t bi = 0; bi < Lo.fbuckets.size(); ++bi)
            if (Lo.fbuckets[bi].own) {
                ++nown;
                Lo.own_uni = (int32_t)bi;
            }
        if (nown != 1 || !Lo.own_sliced) Lo.own_uni = -1;
    }
    if (Lo.own && Lo.own_uni >= 0) {
        // one owner bucket: grouped, padded, interleaved records (owner_grp_kernel)
        // 16-byte gathers: 4 fp32 / 2 fp64 points per thread; threads per variable (FFSAT_OWN_LANES 2, 4 or 8)
        // single-point plans (batch_ref <= 4): one thread per (variable, point), a warp over 32 variables, x read in
        // place (1-point slices) -- no lane idles for want of points
        const bool single = batch_ref <= 4;
        Lo.own_ppt = single ? 1 : precision == 64 ? 2 : 4;
        Lo.own_lanes = single ? 1 : kOwnLanes;
        if (const char* e = std::getenv("FFSAT_OWN_PPT")) Lo.own_ppt = std::atoi(e) == 2 ? 2 : Lo.own_ppt;
        if (const char* e = std::getenv("FFSAT_OWN_LANES")) {
            const int v = std::atoi(e);
            Lo.own_lanes = v == 1 || v == 2 || v == 4 ? v : 8;
        }
        // one-warp CTAs: a CTA's SM slot is released as soon as its group ends, not when the slowest of several
        // groups does (c5 owner kernel 0.94 ms at 8 warps per CTA, 0.88 at 4, 0.85 at 2, 0.81 at 1)
        Lo.own_wpb = 1;
        if (const char* e = std::getenv("FFSAT_OWN_WPB")) {
            const int w = std::atoi(e);
            Lo.own_wpb = w == 8 || w == 4 || w == 2 ? w : 1;
        }
        if (Lo.own_lanes == 1) Lo.own_ppt = 1;
        else if (Lo.own_ppt == 1) Lo.own_ppt = 2;
        const int G = 32 / Lo.own_lanes, NS = 8 * G;   // variable slots per group (warp) and per block
        const FastBucket& b = Lo.fbuckets[(size_t)Lo.own_uni];
        const int64_t n = F.n, nblk = (n + NS - 1) / NS;
        std::vector<int64_t> offA((size_t)n + 1, 0), offB((size_t)n + 1, 0);
        for (int64_t p = b.pos_begin; p < b.pos_end; ++p) {
            const uint32_t* wr = &Lo.fast_words[(size_t)(b.word_off + (p - b.pos_begin) * b.kp)];
            for (int i = 0; i < b.k; ++i) (i == 0 ? offA : offB)[(size_t)(wr[i] & 0x7fffffffu) + 1]++;
        }
        for (int64_t v = 0; v < n; ++v) {
            offA[(size_t)v + 1] += offA[(size_t)v];
            offB[(size_t)v + 1] += offB[(size_t)v];
        }
        std::vector<std::array<uint32_t, 4>> recA((size_t)offA[(size_t)n]), recB((size_t)offB[(size_t)n]);
        {
            std::vector<int64_t> ca(offA.begin(), offA.end() - 1), cb(offB.begin(), offB.end() - 1);
            for (int64_t p = b.pos_begin; p < b.pos_end; ++p) {
                if (p > INT32_MAX) throw Error(FFSAT_ERR_ARG, "formula too large for 32-bit owner records");
                const uint32_t* wr = &Lo.fast_words[(size_t)(b.word_off + (p - b.pos_begin) * b.kp)];
                for (int i = 0; i < b.k; ++i) {
                    const uint32_t v = wr[i] & 0x7fffffffu;
                    std::array<uint32_t, 4> r{(uint32_t)p, 0u, 0u, wr[i] >> 31};
                    int q = 1;
                    for (int j = 0; j < b.k; ++j)
                        if (j != i) r[(size_t)q++] = wr[j];
                    (i == 0 ? recA[(size_t)ca[v]++] : recB[(size_t)cb[v]++]) = r;
                }
            }
        }
        Lo.grp_var.assign((size_t)(nblk * NS), -1);
        Lo.grp_desc.assign((size_t)(nblk * 8 * 4), 0);
        Lo.grp_rec.clear();
        Lo.grp_rec.reserve((size_t)(Lo.n_own_lits * 4 * 5 / 4));
        auto cntA = [&](int32_t v) { return v < 0 ? 0 : offA[(size_t)v + 1] - offA[(size_t)v]; };
        auto cntB = [&](int32_t v) { return v < 0 ? 0 : offB[(size_t)v + 1] - offB[(size_t)v]; };
        // windows of 8 blocks: the window's variables sorted by occurrence counts and dealt in that order to its
        // blocks and groups, so a group's lists, and a block's groups, have about equal lengths (little padding; no
        // warp of a block idles at its barrier) -- the cheapest (padded rows) of three orders: by total count, by
        // literal-0 count, by the other count.  (Slots past n: -1, sorted last.)
        std::vector<int32_t> win_order, o;
        for (int64_t blk = 0; blk < nblk; ++blk) {
            if (blk % 8 == 0) {
                const int64_t wb = std::min<int64_t>(8, nblk - blk) * NS;
                int64_t best_cost = -1;
                o.assign((size_t)wb, -1);
                for (int key = 0; key < 3; ++key) {
                    for (int64_t s = 0; s < wb; ++s) o[(size_t)s] = blk * NS + s < n ? (int32_t)(blk * NS + s) : -1;
                    auto kf = [&](int32_t v) {
                        if (v < 0) return (int64_t)-1;
                        return key == 0 ? cntA(v) + cntB(v) : key == 1 ? (cntA(v) << 24) + cntB(v) : (cntB(v) << 24) + cntA(v);
                    };
                    std::stable_sort(o.begin(), o.end(), [&](int32_t x, int32_t y) { return kf(x) > kf(y); });
                    int64_t cost = 0;
                    for (int64_t g = 0; g < wb / G; ++g) {
                        int64_t la = 0, lb = 0;
                        for (int s = 0; s < G; ++s) {
                            la = std::max(la, cntA(o[(size_t)(G * g + s)]));
                            lb = std::max(lb, cntB(o[(size_t)(G * g + s)]));
                        }
                        cost += la + lb;
                    }
                    if (best_cost < 0 || cost < best_cost) {
                        best_cost = cost;
                        win_order = o;
                    }
                }
            }
            for (int g = 0; g < 8; ++g) {
                const int32_t* grp = &win_order[(size_t)((blk % 8) * NS + g * G)];
                int64_t la = 0, lb = 0;
                for (int s = 0; s < G; ++s) {
                    Lo.grp_var[(size_t)(blk * NS + g * G + s)] = grp[s];
                    la = std::max(la, cntA(grp[s]));
                    lb = std::max(lb, cntB(grp[s]));
                }
                if (la + lb > INT32_MAX) throw Error(FFSAT_ERR_ARG, "variable occurs too often for owner records");
                const uint64_t off = Lo.grp_rec.size() / 4;
                uint32_t* d = &Lo.grp_desc[(size_t)((blk * 8 + g) * 4)];
                d[0] = (uint32_t)off; d[1] = (uint32_t)(off >> 32); d[2] = (uint32_t)la; d[3] = (uint32_t)lb;
                for (int sec = 0; sec < 2; ++sec) {
                    const int64_t rows = sec == 0 ? la : lb;
                    for (int64_t j = 0; j < rows; ++j)
                        for (int s = 0; s < G; ++s) {
                            const int32_t v = grp[s];
                            std::array<uint32_t, 4> r{0u, 0u, 0u, 2u};   // pad
                            if (sec == 0 && j < cntA(v)) r = recA[(size_t)(offA[(size_t)v] + j)];
                            if (sec == 1 && j < cntB(v)) r = recB[(size_t)(offB[(size_t)v] + j)];
                            Lo.grp_rec.insert(Lo.grp_rec.end(), r.begin(), r.end());
                        }
                }
            }
        }
        // 8 pad rows past the last group: the kernel's batches of <= 4 rows, and the next batch it prefetches, read
        // (and mask) past a section's end
        for (int i = 0; i < 8 * G; ++i) Lo.grp_rec.insert(Lo.grp_rec.end(), {0u, 0u, 0u, 2u});
    } else if (Lo.own) {
        if (Lo.fbuckets.size() > 0xffffff) throw Error(FFSAT_ERR_ARG, "too many fast buckets");
        Lo.own_off.assign((size_t)F.n + 1, 0);
        for (const FastBucket& b : Lo.fbuckets)
            if (b.own)
                for (int64_t p = b.pos_begin; p < b.pos_end; ++p)
                    for (int i = 0; i < b.k; ++i)
                        Lo.own_off[(size_t)(Lo.fast_words[(size_t)(b.word_off + (p - b.pos_begin) * b.kp + i)] & 0x7fffffffu) + 1]++;
        for (int32_t v = 0; v < F.n; ++v) Lo.own_off[(size_t)v + 1] += Lo.own_off[(size_t)v];
        Lo.own_rec.assign((size_t)(4 * Lo.n_own_lits), 0);
        std::vector<int64_t> cur(Lo.own_off.begin(), Lo.own_off.end() - 1);
        for (size_t bi = 0; bi < Lo.fbuckets.size(); ++bi) {
            const FastBucket& b = Lo.fbuckets[bi];
            if (!b.own) continue;
            for (int64_t p = b.pos_begin; p < b.pos_end; ++p) {
                const uint32_t* wr = &Lo.fast_words[(size_t)(b.word_off + (p - b.pos_begin) * b.kp)];
                for (int i = 0; i < b.k; ++i) {
                    const uint32_t v = wr[i] & 0x7fffffffu;
                    const int64_t o = cur[v]++;
                    if (p > INT32_MAX) throw Error(FFSAT_ERR_ARG, "formula too large for 32-bit owner records");
                    uint32_t* rec = &Lo.own_rec[(size_t)(4 * o)];
                    rec[0] = (uint32_t)p;
                    int q = 1;
                    for (int j = 0; j < b.k; ++j)
                        if (j != i) rec[q++] = wr[j];
                    while (q < 3) rec[q++] = 0;   // padding (k < 3): never read
                    rec[3] = ((uint32_t)bi << 8) | ((uint32_t)i << 1) | (wr[i] >> 31);
                }
            }
        }
    }

    // ---- T-buffer slots and occurrence CSR (ascending slot order per variable)
    if (path != 2) Lo.tb_fast = 0;
    Lo.tb_slots = Lo.tb_fast + Lo.n_sym_lits;
    std::vector<int32_t> slot_var((size_t)Lo.tb_slots);
    if (path == 2) {
        for (const FastBucket& b : Lo.fbuckets)
            if (!b.own)
            for (int64_t p = b.pos_begin; p < b.pos_end; ++p)
                for (int i = 0; i < b.k; ++i)
                    slot_var[(size_t)(b.slot_off + (p - b.pos_begin) * b.k + i)] =
                        (int32_t)(Lo.fast_words[(size_t)(b.word_off + (p - b.pos_begin) * b.kp + i)] & 0x7fffffffu);
    }
    for (int64_t j = 0; j < Lo.n_sym_lits; ++j) slot_var[(size_t)(Lo.tb_fast + j)] = (int32_t)(Lo.sym_words[(size_t)j] & 0x7fffffffu);
    Lo.occ_off.assign((size_t)F.n + 1, 0);
    for (int32_t v : slot_var) Lo.occ_off[(size_t)v + 1]++;
    for (int32_t v = 0; v < F.n; ++v) Lo.occ_off[(size_t)v + 1] += Lo.occ_off[(size_t)v];
    Lo.occ_slot.assign((size_t)Lo.tb_slots, 0);
    {
        std::vector<int64_t> cur(Lo.occ_off.begin(), Lo.occ_off.end() - 1);
        for (int64_t s = 0; s < Lo.tb_slots; ++s) Lo.occ_slot[(size_t)cur[(size_t)slot_var[(size_t)s]]++] = s;
    }


    // ---- work units: tiled = the classes; global = runs of one bucket with <= 512 literals
    if (path == 1) {
        // wide variant: fp32, every fast bucket one product channel with one shared k <= 16, n small enough
        bool uniform = !Lo.fbuckets.empty();
        for (const FastBucket& b : Lo.fbuckets) {
            const int nch = (b.gA != 0) + (b.gB != 0) + (b.gX != 0);
            uniform = uniform && nch == 1 && b.k <= 16 && b.k == Lo.fbuckets[0].k;
        }
        Lo.wide = allow_wide && precision == 32 && uniform && F.n <= wide_max_n();
        Lo.tmem = Lo.wide && allow_tmem && F.n <= kTmemMaxN && kClassCap <= 16;
        auto red_of = [](int variant) {
            return variant == V_OR || variant == V_NOR ? 1 : variant == V_AND || variant == V_NAND ? 2
                 : variant == V_XOR || variant == V_XNOR ? 3 : 0;
        };
        Lo.wide_red = Lo.fbuckets.empty() ? 0 : red_of(Lo.fbuckets[0].variant);
        for (const FastBucket& b : Lo.fbuckets)
            if (red_of(b.variant) != Lo.wide_red) Lo.wide_red = 0;
        const uint32_t pitch = Lo.wide ? (uint32_t)kWidePitch : (uint32_t)kTilePitch;
        Lo.tiled_words.assign(Lo.fast_words.size(), 0);
        for (size_t i = 0; i < Lo.fast_words.size(); ++i) {
            uint32_t w = Lo.fast_words[i];
            Lo.tiled_words[i] = (w & 0x7fffffffu) * pitch | (w & 0x80000000u);
        }
    }
    // global units hold <= cap literals: 512 for large formulas, smaller for small ones so that the chunk split
    // (<= one chunk per unit) still yields enough CTAs per point tile to fill the GPU
    int64_t gmax = 512;   // FFSAT_GLOBAL_UNIT: tuning override of the largest global unit (literals)
    if (const char* e = std::getenv("FFSAT_GLOBAL_UNIT")) gmax = std::max(16, std::atoi(e));
    const int64_t gcap = std::min<int64_t>(gmax, std::max<int64_t>(32, Lo.n_fast_lits / 1024));
    for (size_t bi = 0; bi < Lo.fbuckets.size(); ++bi) {
        const FastBucket& b = Lo.fbuckets[bi];
        int64_t p = b.pos_begin;
        while (p < b.pos_end) {
            int64_t q = p + 1;
            if (path == 1) {
                while (q < b.pos_end && fast_class[(size_t)q] == fast_class[(size_t)p]) ++q;
            } else {
                q = std::min(b.pos_end, p + std::max<int64_t>(1, gcap / b.k));
            }
            Lo.units.push_back({(int32_t)bi, (int32_t)(q - p), p});
            Lo.unit_rows.push_back((q - p) * b.k);
            p = q;
        }
    }
    return Lo;
}

}  // namespace ffsat
