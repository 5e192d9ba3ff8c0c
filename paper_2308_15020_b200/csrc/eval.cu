// eval.cu -- batch planning of ffsat_eval (chunk split of the fast kernels, scratch sizing).
#include <algorithm>

#include "ctx.hpp"

namespace ffsat {

namespace {
// Pick the number of clause chunks so (point tiles x chunks) fills whole waves of CTAs.
int pick_chunks(int64_t point_tiles, int ctas_per_sm, int num_sm, int64_t n_units) {
    if (n_units <= 0) return 0;
    const int64_t slots = (int64_t)num_sm * std::max(1, ctas_per_sm);
    int best = 1;
    double best_eff = -1;
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

void plan(ffsat_ctx* c, int64_t B) {
    if (c->plan_B == B) return;
    const Layout& L = c->Lo;
    const size_t es = c->esize;
    const int64_t PT = L.wide ? (B + 63) / 64 : (B + 31) / 32;
    int cps = 8;
    if (L.path == 1) {
        c->tiled_smem = L.wide ? wide_smem_bytes(L.n) : tiled_smem_bytes(L.n, L.precision);
        cps = std::max(1, (int)std::min<size_t>(8, (228 * 1024) / (c->tiled_smem + (L.precision == 64 ? 4352 : 2304) + 1024)));
    }
    const int64_t n_units = (int64_t)L.units.size();
    c->n_chunks = L.n_fast > 0 ? pick_chunks(PT, cps, c->num_sm, n_units) : 0;
    // balanced contiguous unit ranges by literal rows
    std::vector<int32_t> cu((size_t)c->n_chunks + 1, 0);
    if (c->n_chunks > 0) {
        int64_t total = 0;
        for (int64_t r : L.unit_rows) total += r;
        int64_t acc = 0;
        int j = 1;
        for (int64_t u = 0; u < n_units && j < c->n_chunks; ++u) {
            acc += L.unit_rows[(size_t)u];
            while (j < c->n_chunks && acc * c->n_chunks >= total * j) cu[j++] = (int32_t)(u + 1);
        }
        for (; j <= c->n_chunks; ++j) cu[j] = (int32_t)n_units;
        cu[c->n_chunks] = (int32_t)n_units;
    }
    upload(c->chunk_units, cu);
    const int64_t parts = std::max<int64_t>(1, c->n_chunks);
    if (L.path == 1) c->P.ensure(std::max<size_t>(16, (size_t)c->n_chunks * L.n * B * es));
    if (L.path == 2 || L.sym_lane) c->xT.ensure(std::max<size_t>(16, (size_t)L.n * B * es));
    c->Tb.ensure(std::max<size_t>(16, (size_t)L.tb_slots * B * es));
    c->fpart.ensure((size_t)parts * B * 8);
    c->upart.ensure((size_t)parts * B * 4);
    c->fsym.ensure(std::max<size_t>(16, (size_t)L.n_sym * B * 8));
    c->usym.ensure(std::max<size_t>(16, (size_t)L.n_sym * B * 4));
    if (L.path == 1) {
        if (L.precision == 64) set_tiled_smem<double>(c->tiled_smem);
        else set_tiled_smem<float>(c->tiled_smem);
        if (L.wide) set_wide_smem(c->tiled_smem);
    }
    c->plan_B = B;
}


}  // namespace ffsat
