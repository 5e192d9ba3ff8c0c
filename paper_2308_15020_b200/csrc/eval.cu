// eval.cu -- launch planning of ffsat_eval: the batch-independent chunk split of the fast kernels (at load) and the
// per-batch scratch sizing.
#include <algorithm>
#include <cstdlib>

#include "ctx.hpp"

namespace ffsat {

namespace {
// Pick the number of clause chunks so (point tiles x chunks) fills whole waves of CTAs.
int pick_chunks(int64_t point_tiles, int ctas_per_sm, int num_sm, int64_t n_units) {
    if (n_units <= 0) return 0;
    const int64_t slots = (int64_t)num_sm * std::max(1, ctas_per_sm);
    int best = 1;
    double best_eff = -1;
    if (const char* e = std::getenv("FFSAT_WAVES")) {   // tuning override: exactly this many waves of CTAs
        const int64_t nc = std::max<int64_t>(1, (std::max(1, std::atoi(e)) * slots) / point_tiles);
        return (int)std::min<int64_t>(nc, n_units);
    }
    for (int w = 1; w <= 4; ++w) {
        int64_t nc = std::max<int64_t>(1, (w * slots) / point_tiles);
        nc = std::min<int64_t>(nc, n_units);
        int64_t ctas = nc * point_tiles;
        int64_t waves = (ctas + slots - 1) / slots;
        double eff = (double)ctas / (double)(waves * slots);
        if (eff > best_eff + 0.05) {
            best_eff = eff;
            best = (int)nc;
        }
        if (eff >= 0.9) break;
    }
    return best;
}

}  // namespace

void plan_chunks(ffsat_ctx* c) {
    const Layout& L = c->Lo;
    const int64_t B = std::max<int64_t>(1, c->batch_ref);   // the reference batch: the split never sees a call's B
    const int64_t PT = L.wide ? (B + 63) / 64 : (B + 31) / 32;
    int cps = 8;
    if (L.path == 1) {
        c->tiled_smem = L.tmem ? tmem_smem_bytes(L.n) : L.wide ? wide_smem_bytes(L.n) : tiled_smem_bytes(L.n, L.precision);
        cps = L.tmem ? 1   // one CTA per SM: 16 warps, the TMEM allocation
                     : std::max(1, (int)std::min<size_t>(8, (228 * 1024) / (c->tiled_smem + (L.precision == 64 ? 4352 : 2304) + 1024)));
    }
    const int64_t n_units = (int64_t)L.units.size();
    // global path: units grouped by length class (buckets ascend in k, so each group is a contiguous unit range):
    // k <= 4, 4 < k <= 16, k > 16 -- each group gets its own chunks and launch (register bound per class)
    int64_t ug[4] = {0, n_units, n_units, n_units};
    if (L.path == 2) {
        auto kof = [&](int64_t u) { return L.fbuckets[(size_t)L.units[(size_t)u].bucket].k; };
        int64_t u = 0;
        // owner-computes buckets (the shortest, a prefix of the units) take no fast-kernel pass: owner_grad_kernel
        // forms their terms per variable
        while (u < n_units && L.fbuckets[(size_t)L.units[(size_t)u].bucket].own) ++u;
        ug[0] = u;
        while (u < n_units && kof(u) <= 4) ++u;
        ug[1] = u;
        while (u < n_units && kof(u) <= 16) ++u;
        ug[2] = u;
        // a small 4 < k <= 16 group runs in the long kernel (any k <= 64): a launch of its own would be latency-bound
        int64_t lits1 = 0;
        for (int64_t q = ug[1]; q < ug[2]; ++q) lits1 += L.unit_rows[(size_t)q];
        if (lits1 < 65536) ug[2] = ug[1];
    }
    int ncg[3] = {0, 0, 0};
    if (L.n_fast > 0) {
        int gcps = cps;   // FFSAT_GLOBAL_CPS: tuning override of the CTAs-per-SM target of the k <= 16 global kernel
        if (const char* e = std::getenv("FFSAT_GLOBAL_CPS")) if (L.path == 2) gcps = std::max(1, std::atoi(e));
        ncg[0] = pick_chunks(PT, gcps, c->num_sm, ug[1] - ug[0]);
        ncg[1] = pick_chunks(PT, gcps, c->num_sm, ug[2] - ug[1]);
        ncg[2] = pick_chunks(PT, 6, c->num_sm, ug[3] - ug[2]);   // long kernel: 32 KB smem per CTA
    }
    c->gchunk[0] = 0;
    for (int g = 0; g < 3; ++g) c->gchunk[g + 1] = c->gchunk[g] + ncg[g];
    c->n_chunks = c->gchunk[3];
    // balanced contiguous unit ranges by literal rows, within each group
    std::vector<int32_t> cu((size_t)c->n_chunks + 1, 0);
    auto split = [&](int64_t ua, int64_t ub, int nc, int j0) {
        int64_t total = 0;
        for (int64_t u = ua; u < ub; ++u) total += L.unit_rows[(size_t)u];
        int64_t acc = 0;
        int j = 1;
        for (int64_t u = ua; u < ub && j < nc; ++u) {
            acc += L.unit_rows[(size_t)u];
            while (j < nc && acc * nc >= total * j) cu[(size_t)(j0 + j++)] = (int32_t)(u + 1);
        }
        for (; j <= nc; ++j) cu[(size_t)(j0 + j)] = (int32_t)ub;
        cu[(size_t)j0] = (int32_t)ua;
    };
    for (int g = 0; g < 3; ++g)
        if (ncg[g] > 0) split(ug[g], ug[g + 1], ncg[g], c->gchunk[g]);
    if (L.tmem && ncg[0] > 0) {
        // the TMEM kernel keeps its chunk's class data (headers, literal words, weights) resident in shared memory
        // after the x tile: more chunks until the largest fits (228 KB per CTA minus the tile and the static part)
        auto res_bytes = [&](int64_t ua, int64_t ub) -> size_t {
            if (ua >= ub) return 0;
            auto wb = [&](int64_t u) {
                const WorkUnit& w = L.units[(size_t)u];
                const FastBucket& b = L.fbuckets[(size_t)w.bucket];
                return b.word_off + (w.pos_begin - b.pos_begin) * b.kp;
            };
            const WorkUnit& wl = L.units[(size_t)ub - 1];
            const int64_t words = wb(ub - 1) + (int64_t)wl.count * L.fbuckets[(size_t)wl.bucket].kp - wb(ua);
            const int64_t cons = wl.pos_begin + wl.count - L.units[(size_t)ua].pos_begin;
            return (size_t)(16 * (ub - ua) + 4 * words + 4 * cons);
        };
        const size_t budget = (size_t)227 * 1024 - (size_t)256 * L.n - 1024;
        for (;;) {
            size_t mx = 0;
            for (int j = 0; j < ncg[0]; ++j) mx = std::max(mx, res_bytes(cu[(size_t)j], cu[(size_t)j + 1]));
            if (mx <= budget) {
                c->tiled_smem = std::max(tmem_smem_bytes(L.n), (size_t)256 * L.n + mx);
                break;
            }
            if (ncg[0] >= ug[1] - ug[0]) throw Error(FFSAT_ERR_ARG, "TMEM kernel: a class does not fit in shared memory");
            ncg[0] = (int)std::min<int64_t>(ug[1] - ug[0], (int64_t)ncg[0] * mx / budget + 1);
            c->gchunk[1] = ncg[0];
            c->gchunk[2] = c->gchunk[3] = ncg[0];
            c->n_chunks = ncg[0];
            cu.assign((size_t)c->n_chunks + 1, 0);
            split(ug[0], ug[1], ncg[0], 0);
        }
    }
    upload(c->chunk_units, cu);
    // the fixed f / unsat summation order: rows r = 0 .. R-1 (fast partials, then root-path constraints) summed in
    // f_groups interleaved groups (r mod f_groups), ascending inside a group, groups in order -- the same order in
    // reduce_f_kernel and in the gradient reduction's fused variant, for every batch size
    // owner_grad_kernel's f / unsat partial rows, one per 8-variable tile, folded 256 to a row (fold_rows_kernel);
    // partial row layout: [chunk rows | folded rows | variable-tile rows]
    // the owner kernels' variable tiles (partial f rows): 256 / kOwnSlice variables (sliced) or 8 (unsliced)
    c->n_vtiles = !L.own ? 0 : L.own_uni >= 0 ? (L.n + 32 * L.own_wpb / L.own_lanes - 1) / (32 * L.own_wpb / L.own_lanes)
                 : L.own_sliced ? (L.n + 256 / kOwnSlice - 1) / (256 / kOwnSlice) : (L.n + 7) / 8;
    c->n_fold = (c->n_vtiles + 255) / 256;
    const int64_t rows = (L.n_fast > 0 ? c->n_chunks + c->n_fold : 0) + L.n_sym;
    c->f_groups = rows > 256 ? 32 : 8;
    {   // root splits: per-class partial regions (S = 1 everywhere if they would exceed 4 GiB at the reference batch)
        const size_t ncl = L.sym_classes.size();
        c->sym_S.assign(ncl, 1);
        c->sym_offT.assign(ncl, 0);
        c->sym_offF.assign(ncl, 0);
        int64_t tT = 0, tF = 0;
        for (size_t i = 0; i < ncl; ++i) {
            const SymClass& cl = L.sym_classes[i];
            if (cl.S <= 1) continue;
            c->sym_S[i] = cl.S;
            c->sym_offT[i] = tT;
            c->sym_offF[i] = tF;
            tT += (int64_t)cl.S * (cl.lit_end - cl.lit_begin);
            tF += (int64_t)cl.S * (cl.end - cl.begin);
        }
        if ((size_t)(tT * (int64_t)c->esize + tF * 8) * (size_t)B > (size_t)4 << 30) {
            c->sym_S.assign(ncl, 1);
            tT = tF = 0;
        }
        c->sym_totT = tT;
        c->sym_totF = tF;
    }
    if (L.path == 1) {
        if (L.tmem) set_tmem_smem(c->tiled_smem);
        else if (L.wide) set_wide_smem(c->tiled_smem);
        else if (L.precision == 64) set_tiled_smem<double>(c->tiled_smem);
        else set_tiled_smem<float>(c->tiled_smem);
    }
    if (ncg[2] > 0) {
        if (L.precision == 64) set_long_smem<double>();
        else set_long_smem<float>();
    }
}

void ensure_scratch(const ffsat_ctx* c, Scratch& S, int64_t B) {
    if (S.B >= B) return;   // buffers sized for a larger batch serve every smaller one (row strides are the call's B)
    const Layout& L = c->Lo;
    const size_t es = c->esize, b = (size_t)B;
    const size_t parts = (size_t)std::max<int64_t>(1, c->n_chunks + c->n_fold + c->n_vtiles);
    if (L.path == 1) S.P.ensure(std::max<size_t>(16, parts * L.n * b * es));
    if (L.path == 2 || L.sym_lane) S.xT.ensure(std::max<size_t>(16, (size_t)L.n * ((b + kOwnSliceMax - 1) / kOwnSliceMax * kOwnSliceMax) * es));   // (sliced: whole slices)
    S.Tb.ensure(std::max<size_t>(16, (size_t)L.tb_slots * b * es));
    S.fpart.ensure(parts * b * 8);
    S.upart.ensure(parts * b * 4);
    S.fsym.ensure(std::max<size_t>(16, (size_t)L.n_sym * b * 8));
    S.usym.ensure(std::max<size_t>(16, (size_t)L.n_sym * b * 4));
    S.TbS.ensure(std::max<size_t>(16, (size_t)c->sym_totT * b * es));
    S.fS.ensure(std::max<size_t>(16, (size_t)c->sym_totF * b * 8));
    S.tree_ctr.ensure(std::max<size_t>(16, L.sym_classes.size() * 4));
    S.B = B;
}


}  // namespace ffsat
