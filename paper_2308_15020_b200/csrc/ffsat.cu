// ffsat.cu -- libffsat.so: context, device layout, launch orchestration and the C-ABI of include/ffsat.h.
// Every compute step runs in the kernels of kernels_eval.cuh / kernels_solve.cuh; the host only parses,
// lays out data (A1-A3) and enqueues launches.  No CPU fallback exists: without a CUDA device every
// compute entry point fails with FFSAT_ERR_CUDA / FFSAT_ERR_ARG.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/ffsat.h"
#include "host.hpp"
#include "ctx.hpp"
#include "kernels_solve.cuh"

using namespace ffsat;

namespace {

thread_local std::string g_err;

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

struct ffsat_search {
    ffsat_ctx* ctx = nullptr;
    int64_t B = 0, point0 = 0;
    uint64_t seed = 0;
    ffsat_solve_params P{};
    DBuf X, Xp, Gx, Gp, fX, fP, dot, eta, done, iters, unsatP, solved, sol, unsat, U, stats, xT;
    DBuf W;                       // this search's current weights (position order, context dtype): ERWA state
    DBuf umax;                    // max U_c of the ERWA update
    DBuf Xm, Y, fy, tmom, phase;  // FISTA state (P.accel = 1): x_{k-1}, y, f(y), momentum t, phase
    Scratch sc;                   // this search's evaluation scratch (referenced by its captured graph)
    int64_t round = 0, iters_issued = 0;
    // one CLS iteration captured as a CUDA graph (replayed by ffsat_search_iterate), in two variants: [1] with the
    // fused check of the trial points (every check_every-th iteration of a round), [0] without
    cudaStream_t cap_stream = nullptr;
    cudaGraphExec_t iter_exec[2] = {nullptr, nullptr};
    int64_t iter_kernels[2] = {0, 0};   // kernels in one captured iteration (launch accounting)
    bool graph_failed = false;
    ~ffsat_search() {
        for (cudaGraphExec_t& g : iter_exec)
            if (g) cudaGraphExecDestroy(g);
        if (cap_stream) cudaStreamDestroy(cap_stream);
    }
    bool checked_next() const { return (iters_issued + 1) % P.check_every == 0; }
};

namespace {

// ------------------------------------------------------------------------------------------------ setup

void upload_layout(ffsat_ctx* c) {
    const Layout& L = c->Lo;
    const bool f64 = L.precision == 64;
    c->esize = f64 ? 8 : 4;
    upload(c->fast_words, L.fast_words);
    if (L.path == 1) upload(c->tiled_words, L.tiled_words);
    std::vector<dev::UnitDev> units;
    for (const WorkUnit& u : L.units) {
        const FastBucket& b = L.fbuckets[(size_t)u.bucket];
        const int64_t wb = b.word_off + (u.pos_begin - b.pos_begin) * b.kp;
        if (u.count > 0xffff || b.kp > 0x7fff || u.pos_begin > INT32_MAX || wb > INT32_MAX)
            throw Error(FFSAT_ERR_ARG, "formula too large for 32-bit work-unit headers");
        units.push_back({u.bucket, u.count | (b.kp << 16), (int32_t)u.pos_begin, (int32_t)wb});
    }
    upload(c->units, units);
    std::vector<dev::FastBucketDev> bks;
    for (const FastBucket& b : L.fbuckets) {
        dev::FastBucketDev d{};
        d.k = b.k; d.kp = b.kp; d.pos_begin = b.pos_begin; d.word_off = b.word_off; d.slot_off = b.slot_off;
        d.g0 = b.g0;
        int ch = 0;
        if (b.gA != 0) { d.c0[ch] = 0.5; d.c1[ch] = 0.5; d.g[ch] = b.gA; ++ch; }   // A: (1 + l)/2
        if (b.gB != 0) { d.c0[ch] = 0.5; d.c1[ch] = -0.5; d.g[ch] = b.gB; ++ch; }  // B: (1 - l)/2
        if (b.gX != 0) { d.c0[ch] = 0.0; d.c1[ch] = 1.0; d.g[ch] = b.gX; ++ch; }   // X: l
        d.nch = ch;
        d.tmin = b.rule.tmin; d.tmax = b.rule.tmax; d.parity = b.rule.parity;
        switch (b.variant) {
        case V_OR: d.red = 1; break;
        case V_NOR: d.red = 1 + 4; break;
        case V_AND: d.red = 2; break;
        case V_NAND: d.red = 2 + 4; break;
        case V_XOR: d.red = 3; break;
        case V_XNOR: d.red = 3 + 4; break;
        default: d.red = 0;
        }
        bks.push_back(d);
    }
    upload(c->buckets, bks);
    upload(c->sym_words, L.sym_words);
    upload(c->sym_off, L.sym_off);
    upload(c->sym_sig, L.sym_sig);
    std::vector<dev::SymSigDev> sg;
    for (const SymSig& s : L.sigs) sg.push_back({s.k, s.Mp, s.tmin, s.tmax, s.parity, 0, s.coef_off, s.g0});
    upload(c->sigs, sg);
    if (f64) upload(c->coef, L.coef);
    else {
        std::vector<float> cf(L.coef.begin(), L.coef.end());
        upload(c->coef, cf);
    }
    upload(c->occ_off, L.occ_off);
    if (L.tb_slots > INT32_MAX) throw Error(FFSAT_ERR_ARG, "too many literal slots");
    std::vector<int32_t> occ(L.occ_slot.begin(), L.occ_slot.end());
    upload(c->occ_slot, occ);
    if (f64) upload(c->w_pos, L.w_pos);
    else {
        std::vector<float> w(L.w_pos.begin(), L.w_pos.end());
        upload(c->w_pos, w);
    }
    upload(c->w_static_orig, c->F.weight);
    if (L.own && L.own_uni >= 0) {
        upload(c->grp_desc, L.grp_desc);
        upload(c->grp_var, L.grp_var);
        upload(c->grp_rec, L.grp_rec);
    } else if (L.own) {
        upload(c->own_off, L.own_off);
        upload(c->own_rec, L.own_rec);
    }
    upload(c->order, L.order);
    // unified position-order CSR for the exact check kernel
    std::vector<int64_t> off{0};
    std::vector<uint32_t> words;
    std::vector<int32_t> rule;
    const Formula& F = c->F;
    for (int64_t p = 0; p < L.m; ++p) {
        int64_t oc = L.order[p];
        int k = (int)(F.offsets[oc + 1] - F.offsets[oc]);
        for (int64_t i = F.offsets[oc]; i < F.offsets[oc + 1]; ++i) {
            int32_t lit = F.lits[i];
            words.push_back((uint32_t)((lit > 0 ? lit : -lit) - 1) | (lit < 0 ? 0x80000000u : 0u));
        }
        off.push_back((int64_t)words.size());
        SatRule r = sat_rule(F.kind[oc], k, F.bound[oc]);
        rule.push_back(r.tmin); rule.push_back(r.tmax); rule.push_back(r.parity);
    }
    upload(c->chk_off, off);
    upload(c->chk_words, words);
    upload(c->chk_rule, rule);
    std::vector<int32_t> longs;
    for (int64_t p = 0; p < L.m; ++p)
        if (off[(size_t)p + 1] - off[(size_t)p] > dev::kCheckLong) longs.push_back((int32_t)p);
    c->n_chk_long = (int32_t)longs.size();
    if (!longs.empty()) upload(c->chk_long, longs);
    for (DBuf* d : {&c->fast_words, &c->tiled_words, &c->units, &c->buckets, &c->sym_words, &c->sym_off,
                    &c->sym_sig, &c->sigs, &c->coef, &c->occ_off, &c->occ_slot, &c->w_pos, &c->w_static_orig, &c->order,
                    &c->chk_off, &c->chk_words, &c->chk_rule, &c->chk_long, &c->own_off, &c->own_rec, &c->grp_desc,
                    &c->grp_var, &c->grp_rec})
        c->persistent_bytes += (int64_t)d->bytes;
}

ffsat_ctx* make_ctx(Formula&& F, const ffsat_options* opt) {
    ffsat_options o{0, 0, 0, 0};
    if (opt) o = *opt;
    if (o.batch_ref < 0) throw Error(FFSAT_ERR_ARG, "batch_ref must be >= 0");
    validate(F);
    std::unique_ptr<ffsat_ctx> c(new ffsat_ctx());
    c->F = std::move(F);
    c->Lo = build_layout(c->F, o.path, o.precision, o.batch_ref > 0 ? o.batch_ref : 1024);
    c->device = o.device;
    c->batch_ref = o.batch_ref > 0 ? o.batch_ref : 1024;
    if (o.device >= 0) {
        int ndev = 0;
        cudaError_t e = cudaGetDeviceCount(&ndev);
        if (e != cudaSuccess || ndev == 0) {
            cudaGetLastError();
            throw Error(FFSAT_ERR_CUDA, "no CUDA device available (libffsat has no CPU fallback)");
        }
        if (o.device >= ndev) throw Error(FFSAT_ERR_ARG, "device ordinal out of range");
        CK(cudaSetDevice(o.device));
        CK(cudaDeviceGetAttribute(&c->num_sm, cudaDevAttrMultiProcessorCount, o.device));
        upload_layout(c.get());
        plan_chunks(c.get());
    }
    return c.release();
}

void need_device(const ffsat_ctx* c) {
    if (!c) throw Error(FFSAT_ERR_ARG, "null context");
    if (c->device < 0) throw Error(FFSAT_ERR_ARG, "host-only context (device = -1) cannot compute");
    CK(cudaSetDevice(c->device));
}

// ------------------------------------------------------------------------------------------------ eval

void eval_device(ffsat_ctx* c, const void* x, int64_t B, double* f, void* grad, int32_t* unsat, cudaStream_t st,
                 bool profiled = false, Scratch* scr = nullptr) {
    Scratch& S = scr ? *scr : c->scr;
    if (c->Lo.precision == 64)
        eval_device_t<double>(c, S, (const double*)x, B, f, (double*)grad, unsat, c->w_pos.as<double>(), st, profiled);
    else
        eval_device_t<float>(c, S, (const float*)x, B, f, (float*)grad, unsat, c->w_pos.as<float>(), st, profiled);
}

ffsat_status fail(ffsat_ctx* c, const Error& e) {
    g_err = e.what();
    if (c) c->err = e.what();
    return e.code;
}

ffsat_status fail_std(ffsat_ctx* c, const std::exception& e) {
    g_err = std::string("internal error: ") + e.what();
    if (c) c->err = g_err;
    return FFSAT_ERR_ARG;
}

#define ABI_TRY(ctxp) try {
#define ABI_CATCH(ctxp)                                       \
    }                                                         \
    catch (const Error& e) { return fail(ctxp, e); }          \
    catch (const std::bad_alloc&) { return fail(ctxp, Error(FFSAT_ERR_OOM, "host out of memory")); } \
    catch (const std::exception& e) { return fail_std(ctxp, e); }

int64_t exact_unsat(const Formula& F, const int8_t* a, double* fw) {
    int64_t cnt = 0;
    double w = 0;
    for (int64_t c = 0; c < F.m(); ++c) {
        int k = (int)(F.offsets[c + 1] - F.offsets[c]);
        int t = 0;
        for (int64_t i = F.offsets[c]; i < F.offsets[c + 1]; ++i) {
            int32_t lit = F.lits[i];
            bool var_true = a[(lit > 0 ? lit : -lit) - 1] < 0;
            t += (lit > 0) == var_true;
        }
        SatRule r = sat_rule(F.kind[c], k, F.bound[c]);
        bool sat = t >= r.tmin && t <= r.tmax && (r.parity == 0 || (r.parity == 1) == ((t & 1) == 1));
        if (!sat) {
            ++cnt;
            w += F.weight[c];
        }
    }
    if (fw) *fw = w;
    return cnt;
}

// ------------------------------------------------------------------------------------------------ search

template <typename T>
void search_eval(ffsat_search* s, const void* x, double* f, void* g, int32_t* u, cudaStream_t st) {
    eval_device_t<T>(s->ctx, s->sc, (const T*)x, s->B, f, (T*)g, u, s->W.as<T>(), st, false);
}

void search_alloc(ffsat_search* s) {
    const size_t es = s->ctx->esize, Bn = (size_t)s->B * s->ctx->Lo.n;
    const int64_t B = s->B, m = s->ctx->Lo.m;
    for (DBuf* d : {&s->X, &s->Xp, &s->Gx, &s->Gp}) d->ensure(std::max<size_t>(16, Bn * es));
    for (DBuf* d : {&s->fX, &s->fP, &s->dot, &s->eta}) d->ensure((size_t)B * 8);
    for (DBuf* d : {&s->done, &s->iters, &s->unsatP, &s->solved, &s->unsat}) d->ensure((size_t)B * 4);
    s->sol.ensure(std::max<size_t>(16, Bn));
    s->U.ensure(std::max<size_t>(16, (size_t)m * 4));
    s->W.ensure(std::max<size_t>(16, (size_t)m * es));
    s->umax.ensure(16);
    s->stats.ensure(64);
    if (s->P.accel) {
        for (DBuf* d : {&s->Xm, &s->Y}) d->ensure(std::max<size_t>(16, Bn * es));
        for (DBuf* d : {&s->fy, &s->tmom}) d->ensure((size_t)B * 8);
        s->phase.ensure((size_t)B * 4);
    }
    ensure_scratch(s->ctx, s->sc, B);
    CK(cudaMemset(s->solved.p, 0, (size_t)B * 4));
    CK(cudaMemset(s->unsat.p, 0, (size_t)B * 4));
    CK(cudaMemset(s->U.p, 0, (size_t)std::max<int64_t>(m, 4) * 4));
    CK(cudaMemset(s->done.p, 0, (size_t)B * 4));
}

dev::PgdArgs pgd_args(ffsat_search* s, int mode, bool checked) {
    dev::PgdArgs a{};
    a.B = s->B; a.n = s->ctx->Lo.n; a.eta0 = s->P.eta0; a.eta_min = s->P.eta_min; a.c1 = s->P.armijo_c1;
    a.max_inner = s->P.max_inner; a.X = s->X.p; a.Xp = s->Xp.p; a.Gx = s->Gx.p; a.Gp = s->Gp.p;
    a.fX = s->fX.as<double>(); a.fP = s->fP.as<double>(); a.dot = s->dot.as<double>(); a.eta = s->eta.as<double>();
    a.done = s->done.as<int32_t>(); a.iters = s->iters.as<int32_t>(); a.unsatP = s->unsatP.as<int32_t>();
    a.solved = s->solved.as<int32_t>(); a.sol = s->sol.as<int8_t>(); a.mode = mode; a.checked = checked ? 1 : 0;
    return a;
}

// The (non-fused) PGD step: one CTA per point, 1024 threads when n >= 2048 (the per-point row loop is the latency),
// else 256 -- chosen from n only (batch-independent bits); fp32 follows the gradient reduction programmatically.
void launch_pgd_step(ffsat_search* s, const dev::PgdArgs& a, cudaStream_t st, bool pdl) {
    const bool f64 = s->ctx->Lo.precision == 64, wide = s->ctx->Lo.n >= 2048;
    const dim3 g((unsigned)s->B);
    if (f64) {
        if (wide) dev::pgd_step_kernel<double, 1024><<<g, 1024, 0, st>>>(a);
        else dev::pgd_step_kernel<double, 256><<<g, 256, 0, st>>>(a);
    } else if (pdl) {
        if (wide) launch_pdl(dev::pgd_step_kernel<float, 1024>, g, dim3(1024), 0, st, a);
        else launch_pdl(dev::pgd_step_kernel<float, 256>, g, dim3(256), 0, st, a);
    } else {
        if (wide) dev::pgd_step_kernel<float, 1024><<<g, 1024, 0, st>>>(a);
        else dev::pgd_step_kernel<float, 256><<<g, 256, 0, st>>>(a);
    }
}

dev::FistaArgs fista_args(ffsat_search* s, int mode, bool checked) {
    dev::FistaArgs f{};
    f.p = pgd_args(s, mode, checked);
    f.Xm = s->Xm.p; f.Y = s->Y.p; f.fy = s->fy.as<double>(); f.t = s->tmom.as<double>(); f.phase = s->phase.as<int32_t>();
    return f;
}

// FISTA mode (P.accel = 1): evaluate the point (X at a round start, else Xp) and take the FISTA step; the TMEM path
// fuses the reduction of its point-major partials into the step as pgd_fused_kernel does.
void fista_round_step(ffsat_search* s, int mode, bool checked, cudaStream_t st) {
    ffsat_ctx* c = s->ctx;
    const bool f64 = c->Lo.precision == 64;
    const dev::FistaArgs a = fista_args(s, mode, checked);
    const void* xe = mode == 0 ? s->X.p : s->Xp.p;
    int32_t* u = checked ? s->unsatP.as<int32_t>() : nullptr;
    const unsigned B = (unsigned)s->B;
    if (!f64 && c->Lo.tmem) {
        eval_device_t<float>(c, s->sc, (const float*)xe, s->B, nullptr, nullptr, u, s->W.as<float>(), st, false, true);
        const dev::PmReduce<float> r = pm_reduce_args<float>(c, s->sc, s->B, checked);
        launch_pdl(dev::fista_step_kernel<float, true>, dim3(B), dim3(256), 0, st, a, r);
    } else if (f64) {
        search_eval<double>(s, xe, s->fP.as<double>(), s->Gp.p, u, st);
        dev::fista_step_kernel<double, false><<<B, 256, 0, st>>>(a, dev::PmReduce<double>{});
    } else {
        search_eval<float>(s, xe, s->fP.as<double>(), s->Gp.p, u, st);
        launch_pdl(dev::fista_step_kernel<float, false>, dim3(B), dim3(256), 0, st, a, dev::PmReduce<float>{});
    }
    CK(cudaGetLastError());
}

void search_begin_round(ffsat_search* s, cudaStream_t st) {
    const bool f64 = s->ctx->Lo.precision == 64;
    s->ctx->launches += 1;   // eta / done / iterations are reset by the round-start PGD step itself
    if (s->P.accel) {
        fista_round_step(s, 0, false, st);
        s->iters_issued = 0;
        return;
    }
    // the round's start point x (rephased): f and gradient, no check (the round-end check catches solutions)
    dev::PgdArgs a = pgd_args(s, 0, false);
    if (!f64 && s->ctx->Lo.tmem) {
        eval_device_t<float>(s->ctx, s->sc, s->X.as<float>(), s->B, nullptr, nullptr, nullptr, s->W.as<float>(), st, false, true);
        const dev::PmReduce<float> r = pm_reduce_args<float>(s->ctx, s->sc, s->B, false);
        launch_pdl(dev::pgd_fused_kernel<float>, dim3((unsigned)s->B), dim3(256), 0, st, a, r);
    } else {
        if (f64) search_eval<double>(s, s->X.p, s->fX.as<double>(), s->Gx.p, nullptr, st);
        else search_eval<float>(s, s->X.p, s->fX.as<double>(), s->Gx.p, nullptr, st);
        launch_pgd_step(s, a, st, false);
    }
    CK(cudaGetLastError());
    s->iters_issued = 0;
}

void search_iterate_one(ffsat_search* s, bool checked, cudaStream_t st);

// Capture one iteration of each variant (eval + PGD step, forked root-path streams included) into a graph once per
// search; afterwards each iteration is one cudaGraphLaunch (no per-kernel launch latency on the host or device).
bool search_capture(ffsat_search* s) {
    if (s->iter_exec[0] && s->iter_exec[1]) return true;
    if (s->graph_failed) return false;
    if (!s->cap_stream) CK(cudaStreamCreateWithFlags(&s->cap_stream, cudaStreamNonBlocking));
    // the graphs reference only this search's buffers (sized at create: allocations never happen inside a
    // capture) and the context's persistent layout, which is never reallocated after load
    ensure_scratch(s->ctx, s->sc, s->B);
    s->sc.fk.ensure();
    const int64_t before = s->ctx->launches;
    for (int v = 0; v < 2; ++v) {
        cudaGraph_t g = nullptr;
        if (cudaStreamBeginCapture(s->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
            cudaGetLastError();
            s->graph_failed = true;
            return false;
        }
        const int64_t l0 = s->ctx->launches;
        bool ok = true;
        try {
            search_iterate_one(s, v == 1, s->cap_stream);
        } catch (const Error&) {
            ok = false;
        }
        const cudaError_t e = cudaStreamEndCapture(s->cap_stream, &g);
        s->iter_kernels[v] = s->ctx->launches - l0;
        if (!ok || e != cudaSuccess || !g || cudaGraphInstantiate(&s->iter_exec[v], g, 0) != cudaSuccess) {
            cudaGetLastError();
            if (g) cudaGraphDestroy(g);
            for (cudaGraphExec_t& x : s->iter_exec)
                if (x) { cudaGraphExecDestroy(x); x = nullptr; }
            s->graph_failed = true;
            s->ctx->launches = before;
            return false;
        }
        cudaGraphDestroy(g);
    }
    s->ctx->launches = before;
    return true;
}

void search_iterate(ffsat_search* s, int n_iters, cudaStream_t st) {
    const bool graphs = n_iters > 0 && search_capture(s);
    for (int i = 0; i < n_iters; ++i) {
        const bool chk = s->checked_next();
        if (graphs) {
            CK(cudaGraphLaunch(s->iter_exec[chk ? 1 : 0], st));
            s->ctx->launches += s->iter_kernels[chk ? 1 : 0];
        } else {
            search_iterate_one(s, chk, st);
        }
        s->iters_issued += 1;
    }
}

// One PGD iteration: evaluate the trial points (with the fused check of their rounded assignment when `checked`),
// then the Armijo accept / eta update / next trial point.
void search_iterate_one(ffsat_search* s, bool checked, cudaStream_t st) {
    const bool f64 = s->ctx->Lo.precision == 64;
    if (s->P.accel) {
        s->ctx->launches += 1;
        fista_round_step(s, 1, checked, st);
        return;
    }
    dev::PgdArgs a = pgd_args(s, 1, checked);
    int32_t* u = checked ? s->unsatP.as<int32_t>() : nullptr;
    s->ctx->launches += 1;
    if (!f64 && s->ctx->Lo.tmem) {
        // tiled TMEM path: the evaluation stops at its point-major partials; the PGD step reduces them itself
        eval_device_t<float>(s->ctx, s->sc, s->Xp.as<float>(), s->B, nullptr, nullptr, u, s->W.as<float>(), st, false, true);
        const dev::PmReduce<float> r = pm_reduce_args<float>(s->ctx, s->sc, s->B, checked);
        launch_pdl(dev::pgd_fused_kernel<float>, dim3((unsigned)s->B), dim3(256), 0, st, a, r);
    } else if (f64) {
        search_eval<double>(s, s->Xp.p, s->fP.as<double>(), s->Gp.p, u, st);
        launch_pgd_step(s, a, st, false);
    } else {
        search_eval<float>(s, s->Xp.p, s->fP.as<double>(), s->Gp.p, u, st);
        launch_pgd_step(s, a, st, true);
    }
    CK(cudaGetLastError());
}

void check_kernels(ffsat_search* s, cudaStream_t st);

void search_check(ffsat_search* s, cudaStream_t st) {
    ffsat_ctx* c = s->ctx;
    const Layout& L = c->Lo;
    CK(cudaMemsetAsync(s->unsat.p, 0, (size_t)s->B * 4, st));
    if (L.m > 0) check_kernels(s, st);
    // points whose sgn(x) satisfies every constraint are solved (kept in sol, so a later restart cannot lose them)
    if (L.precision == 64) dev::mark_solved_kernel<double><<<(unsigned)s->B, 128, 0, st>>>(s->X.as<double>(), s->unsat.as<int32_t>(), s->solved.as<int32_t>(), s->sol.as<int8_t>(), L.n);
    else dev::mark_solved_kernel<float><<<(unsigned)s->B, 128, 0, st>>>(s->X.as<float>(), s->unsat.as<int32_t>(), s->solved.as<int32_t>(), s->sol.as<int8_t>(), L.n);
    s->ctx->launches += 1;
    CK(cudaGetLastError());
}

void check_kernels(ffsat_search* s, cudaStream_t st) {
    ffsat_ctx* c = s->ctx;
    const Layout& L = c->Lo;
    CK(cudaMemsetAsync(s->U.p, 0, (size_t)L.m * 4, st));
    // sign words S[pt][v] (32 points per word), then one thread per (constraint, 32 points)
    const int64_t PT = (s->B + 31) / 32;
    s->xT.ensure(std::max<size_t>(16, (size_t)PT * L.n * 4));
    uint32_t* S = s->xT.as<uint32_t>();
    dim3 pg(blocks_for(L.n, 8 * 4), (unsigned)PT);
    if (L.precision == 64) dev::signpack_kernel<double><<<pg, 256, 0, st>>>(s->X.as<double>(), S, s->B, L.n);
    else dev::signpack_kernel<float><<<pg, 256, 0, st>>>(s->X.as<float>(), S, s->B, L.n);
    dev::CheckBitsArgs a{};
    a.S = S; a.B = s->B; a.n = L.n; a.m = L.m; a.off = c->chk_off.as<int64_t>();
    a.words = c->chk_words.as<uint32_t>(); a.rule = c->chk_rule.as<int32_t>();
    a.U = s->U.as<int32_t>(); a.unsat = s->unsat.as<int32_t>();
    if (L.max_k <= 64) {   // short rows: thread per constraint over TPC point tiles (the largest TPC with >= 2 waves)
        const int64_t cx = blocks_for(L.m, 256);
        int tpc = 8;
        while (tpc > 1 && cx * ((PT + tpc - 1) / tpc) < 2 * c->num_sm) tpc >>= 1;
        dim3 grid((unsigned)cx, (unsigned)((PT + tpc - 1) / tpc));
        switch (tpc) {
        case 8: dev::check_rows_kernel<8><<<grid, 256, 0, st>>>(a); break;
        case 4: dev::check_rows_kernel<4><<<grid, 256, 0, st>>>(a); break;
        case 2: dev::check_rows_kernel<2><<<grid, 256, 0, st>>>(a); break;
        default: dev::check_rows_kernel<1><<<grid, 256, 0, st>>>(a); break;
        }
        s->ctx->launches += 2;
        CK(cudaGetLastError());
        return;
    }
    // chunks: about one wave of CTAs, at least 1024 literals each (each CTA stages the tile's sign words)
    const int64_t want = std::max<int64_t>(1, (int64_t)c->num_sm * 8 / PT);
    const int64_t by_work = std::max<int64_t>(1, L.L / 1024);
    const int64_t chunks = std::min<int64_t>(std::min<int64_t>(want, by_work), std::min<int64_t>(65535, (L.m + 255) / 256));
    a.cons_per_cta = (L.m + chunks - 1) / chunks;
    dim3 grid((unsigned)PT, (unsigned)((L.m + a.cons_per_cta - 1) / a.cons_per_cta));
    const size_t tile = (size_t)L.n * 4;
    a.skip_long = c->n_chk_long > 0 ? 1 : 0;
    if (tile <= 96 * 1024) {
        if (tile > 48 * 1024) CK(cudaFuncSetAttribute(dev::check_bits_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile));
        dev::check_bits_kernel<true><<<grid, 256, tile, st>>>(a);
    } else {
        dev::check_bits_kernel<false><<<grid, 256, 0, st>>>(a);
    }
    s->ctx->launches += 2;
    if (c->n_chk_long > 0) {   // the long rows: one warp per (row, 32-point tile)
        dim3 lg((unsigned)PT, (unsigned)((c->n_chk_long + 7) / 8));
        if (tile <= 96 * 1024) {
            if (tile > 48 * 1024) CK(cudaFuncSetAttribute(dev::check_long_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tile));
            dev::check_long_kernel<true><<<lg, 256, tile, st>>>(a, c->chk_long.as<int32_t>(), c->n_chk_long);
        } else {
            dev::check_long_kernel<false><<<lg, 256, 0, st>>>(a, c->chk_long.as<int32_t>(), c->n_chk_long);
        }
        s->ctx->launches += 1;
    }
    CK(cudaGetLastError());
}

int policy_codes(int policy, int* p) {  // 'R' = 0, 'O' = 1, 'F' = 2
    if (policy == 0) { p[0] = 0; p[1] = 1; p[2] = 2; return 3; }   // (ROF)^inf
    if (policy == 1) { p[0] = 0; p[1] = 2; p[2] = 0; return 2; }   // (RF)^inf
    p[0] = 0; p[1] = 0; p[2] = 0;
    return 1;                                                      // R only
}

void search_restart(ffsat_search* s, const int32_t* Ug, cudaStream_t st) {
    const Layout& L = s->ctx->Lo;
    const bool f64 = L.precision == 64;
    const int32_t* U = Ug ? Ug : s->U.as<int32_t>();
    if (s->P.adaptive_weights && L.m > 0) {
        s->ctx->launches += 1;
        const unsigned g = (unsigned)std::min<int64_t>(4 * 148, (L.m + 255) / 256);
        CK(cudaMemsetAsync(s->umax.p, 0, 4, st));
        dev::umax_kernel<<<g, 256, 0, st>>>(U, L.m, s->umax.as<int32_t>());
        if (f64) dev::erwa_kernel<double><<<g, 256, 0, st>>>(s->W.as<double>(), U, L.m, s->P.alpha, s->umax.as<int32_t>());
        else dev::erwa_kernel<float><<<g, 256, 0, st>>>(s->W.as<float>(), U, L.m, s->P.alpha, s->umax.as<int32_t>());
        s->ctx->launches += 1;
    }
    int p[3];
    int len = policy_codes(s->P.policy, p);
    const int64_t tot = s->B * L.n;
    const uint32_t nr = (uint32_t)(s->round + 1);
    if (tot > 0) {
        s->ctx->launches += 1;
        if (f64) dev::rephase_kernel<double><<<blocks_for(tot, 256), 256, 0, st>>>(s->X.as<double>(), s->B, L.n, s->seed, s->point0, nr, len, p[0], p[1], p[2]);
        else dev::rephase_kernel<float><<<blocks_for(tot, 256), 256, 0, st>>>(s->X.as<float>(), s->B, L.n, s->seed, s->point0, nr, len, p[0], p[1], p[2]);
    }
    CK(cudaGetLastError());
    s->round += 1;
}

void search_reduce(ffsat_search* s, cudaStream_t st) {
    s->ctx->launches += 1;
    dev::stats_kernel<<<1, 1024, 0, st>>>(s->done.as<int32_t>(), s->solved.as<int32_t>(), s->unsat.as<int32_t>(), s->B,
                                          s->point0, s->stats.as<int64_t>());
    CK(cudaGetLastError());
}

void search_stats(ffsat_search* s, cudaStream_t st, ffsat_search_stats* out) {
    search_reduce(s, st);
    int64_t h[3];
    CK(cudaMemcpyAsync(h, s->stats.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out->round = s->round;
    out->iterations = s->iters_issued;
    out->active = h[0];
    out->solved_point = h[1] != INT64_MAX ? h[1] : -1;
    out->best_unsat = h[2] != INT64_MAX ? (h[2] >> 32) : -1;
    out->best_point = h[2] != INT64_MAX ? (h[2] & 0xffffffffLL) : -1;
}

void search_assignment(ffsat_search* s, int64_t lp, int8_t* out) {
    const int n = s->ctx->Lo.n;
    int32_t solved = 0;
    CK(cudaMemcpy(&solved, s->solved.as<int32_t>() + lp, 4, cudaMemcpyDeviceToHost));
    if (solved) {
        CK(cudaMemcpy(out, s->sol.as<int8_t>() + lp * n, (size_t)n, cudaMemcpyDeviceToHost));
        return;
    }
    const size_t es = s->ctx->esize;
    std::vector<unsigned char> row((size_t)n * es);
    CK(cudaMemcpy(row.data(), (const char*)s->X.p + lp * n * es, row.size(), cudaMemcpyDeviceToHost));
    for (int v = 0; v < n; ++v) {
        double xv = es == 8 ? ((double*)row.data())[v] : (double)((float*)row.data())[v];
        out[v] = xv < 0 ? -1 : 1;
    }
}

void check_params(const ffsat_solve_params& p) {
    if (!(p.eta0 > 0) || !(p.eta_min >= 0) || !(p.armijo_c1 >= 0 && p.armijo_c1 < 1) || !(p.alpha >= 0 && p.alpha <= 1) ||
        p.max_inner < 1 || p.check_every < 1 || p.policy < 0 || p.policy > 2 || p.accel < 0 || p.accel > 1 || p.reserved != 0)
        throw Error(FFSAT_ERR_ARG, "invalid solve parameters");
}

}  // namespace

// ================================================================================================ C-ABI

extern "C" {

void ffsat_default_params(ffsat_solve_params* p) {
    if (!p) return;
    p->eta0 = 1.0;
    p->eta_min = 1e-12;
    p->armijo_c1 = 1e-4;
    p->alpha = 0.4;
    p->max_inner = 500;
    p->check_every = 10;
    p->policy = 0;
    p->adaptive_weights = 1;
    p->timeout_s = 0;
    p->accel = 0;
    p->reserved = 0;
}

const char* ffsat_version(void) { return "ffsat-b200 1 (sm_100a)"; }

const char* ffsat_last_error(const ffsat_ctx* ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

ffsat_status ffsat_load(const ffsat_formula* f, const ffsat_options* opt, ffsat_ctx** out) {
    ABI_TRY(nullptr)
    if (!f || !out) throw Error(FFSAT_ERR_ARG, "null argument");
    *out = nullptr;
    *out = make_ctx(from_arrays(*f), opt);
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_load_file(const char* path, const ffsat_options* opt, ffsat_ctx** out) {
    ABI_TRY(nullptr)
    if (!path || !out) throw Error(FFSAT_ERR_ARG, "null argument");
    *out = nullptr;
    std::ifstream in(path, std::ios::binary);
    if (!in) throw Error(FFSAT_ERR_ARG, std::string("cannot open ") + path);
    std::stringstream ss;
    ss << in.rdbuf();
    *out = make_ctx(parse_text(ss.str()), opt);
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_info(const ffsat_ctx* c, ffsat_info_t* o) {
    ABI_TRY(nullptr)
    if (!c || !o) throw Error(FFSAT_ERR_ARG, "null argument");
    const Layout& L = c->Lo;
    o->n_vars = L.n; o->precision = L.precision; o->n_cons = L.m; o->n_lits = L.L;
    o->n_fast_cons = L.n_fast; o->n_sym_cons = L.n_sym; o->n_fast_lits = L.n_fast_lits; o->n_sym_lits = L.n_sym_lits;
    o->sym_root_lits = L.sym_root_lits; o->path = L.path; o->wide = L.tmem ? 2 : L.wide ? 1 : 0; o->max_k = L.max_k; o->device_bytes = c->persistent_bytes;
    o->n_own_lits = L.n_own_lits;
    o->n_tree_cons = L.n_tree_cons; o->tree_work = L.tree_work;
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_export(const ffsat_ctx* c, uint8_t* kind, int32_t* bound, double* weight, int64_t* offsets, int32_t* lits) {
    ABI_TRY(nullptr)
    if (!c) throw Error(FFSAT_ERR_ARG, "null context");
    const Formula& F = c->F;
    if (kind) std::copy(F.kind.begin(), F.kind.end(), kind);
    if (bound) std::copy(F.bound.begin(), F.bound.end(), bound);
    if (weight) std::copy(F.weight.begin(), F.weight.end(), weight);
    if (offsets) std::copy(F.offsets.begin(), F.offsets.end(), offsets);
    if (lits) std::copy(F.lits.begin(), F.lits.end(), lits);
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_eval(ffsat_ctx* c, const void* x, int64_t B, int32_t on_device, double* f_out, void* grad_out,
                        int32_t* unsat_out, void* stream) {
    ABI_TRY(c)
    need_device(c);
    if (B < 0 || (B > 0 && (!x || !f_out))) throw Error(FFSAT_ERR_ARG, "bad eval arguments");
    if (B > INT32_MAX / 2) throw Error(FFSAT_ERR_ARG, "batch too large");
    cudaStream_t st = S(stream);
    const size_t es = c->esize;
    if (B == 0) return FFSAT_OK;
    if (on_device) {
        eval_device(c, x, B, f_out, grad_out, unsat_out, st);
        return FFSAT_OK;
    }
    // host buffers: stage, compute, copy back, pipelined in equal chunks of Bc points (the last one padded with
    // zero points) so the H2D copy of chunk i + 1 and the D2H copy of chunk i - 1 overlap the evaluation of chunk
    // i (two copy engines); non-finite coordinates are flagged by a device kernel on the staged copy.
    // 2 chunks, up to 4 for batches over ~2 MB (smaller chunks multiply the tiled path's partial-tile traffic)
    const size_t xbytes = (size_t)B * (size_t)c->Lo.n * es;
    // chunks of at least batch_ref points: the launch plan is sized for batch_ref, a smaller chunk underfills the GPU
    int64_t nchunk = B < 512 ? 1 : xbytes >= (4u << 20) ? 4 : xbytes >= (2u << 20) ? 3 : 2;
    nchunk = std::max<int64_t>(1, std::min<int64_t>(nchunk, B / std::max<int64_t>(1, c->batch_ref)));
    // batches of >= 512 points: two half-batch chunks evaluated CONCURRENTLY on two compute streams, each with its
    // own scratch and side streams (each fills half the GPU; the copies of one overlap the other's evaluation)
    const bool dual = nchunk == 1 && B >= 512;
    if (dual) nchunk = 2;
    // grouped owner path (c5-like: large n, small batches): 9..32 points go as 8-point chunks -- each one 8-point
    // x^T slice at 1 point per thread -- so the H2D copies of the later chunks and the D2H copies of the earlier ones
    // overlap the evaluations (the copies of 2 x 4 n B bytes dominate such a step)
    const int64_t own_q = c->Lo.own_uni >= 0 && c->esize == 4 && c->Lo.own_ppt == 4 && c->Lo.own_lanes == 8 ? 8 : 0;
    const bool ownq = nchunk == 1 && own_q > 0 && B > own_q && B <= 4 * own_q;
    if (ownq) nchunk = (B + own_q - 1) / own_q;
    const int64_t Bc = ownq ? own_q : nchunk == 1 ? B : ((B + nchunk - 1) / nchunk + 63) / 64 * 64;
    const int64_t nck = Bc > 0 ? (B + Bc - 1) / Bc : 0;
    const size_t n = (size_t)c->Lo.n;
    c->x_stage.ensure(std::max<size_t>(16, (size_t)(nck * Bc) * n * es));
    c->f_stage.ensure(std::max<size_t>(16, (size_t)(nck * Bc) * 8));
    c->u_stage.ensure(std::max<size_t>(16, (size_t)(nck * Bc) * 4));
    if (grad_out) c->g_stage.ensure(std::max<size_t>(16, (size_t)(nck * Bc) * n * es));
    c->nf_flag.ensure(16);
    if (!c->copy_h2d) {
        CK(cudaStreamCreateWithFlags(&c->copy_h2d, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->copy_d2h, cudaStreamNonBlocking));
        CK(cudaMallocHost(&c->nf_host, 16));
    }
    if (dual && !c->comp2) CK(cudaStreamCreateWithFlags(&c->comp2, cudaStreamNonBlocking));
    while ((int64_t)c->ev_h2d.size() < nck + 1) {
        cudaEvent_t e1, e2;
        CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
        c->ev_h2d.push_back(e1);
        c->ev_done.push_back(e2);
    }
    char* xs = c->x_stage.as<char>();
    char* gs = c->g_stage.as<char>();
    // the compute stream's prior work is ordered before the copies (ev_done[nck] marks it)
    CK(cudaEventRecord(c->ev_done[(size_t)nck], st));
    CK(cudaStreamWaitEvent(c->copy_h2d, c->ev_done[(size_t)nck], 0));
    CK(cudaMemsetAsync(c->nf_flag.p, 0, 4, c->copy_h2d));
    if (nck * Bc > B) CK(cudaMemsetAsync(xs + (size_t)B * n * es, 0, (size_t)(nck * Bc - B) * n * es, c->copy_h2d));
    for (int64_t i = 0; i < nck; ++i) {
        const int64_t r0 = i * Bc, r1 = std::min(B, r0 + Bc);
        if (r1 > r0 && n) CK(cudaMemcpyAsync(xs + (size_t)r0 * n * es, (const char*)x + (size_t)r0 * n * es, (size_t)(r1 - r0) * n * es,
                                             cudaMemcpyHostToDevice, c->copy_h2d));
        CK(cudaEventRecord(c->ev_h2d[(size_t)i], c->copy_h2d));
    }
    if (dual) {
        ensure_scratch(c, c->scr, Bc);
        ensure_scratch(c, c->scr2, Bc);
    }
    for (int64_t i = 0; i < nck; ++i) {
        const int64_t r0 = i * Bc, r1 = std::min(B, r0 + Bc);
        cudaStream_t cs = dual && i == 1 ? c->comp2 : st;
        CK(cudaStreamWaitEvent(cs, c->ev_h2d[(size_t)i], 0));   // (also orders comp2 after st's prior work)
        const size_t cnt = (size_t)Bc * n;
        if (cnt) {
            if (es == 8) dev::nonfinite_kernel<double><<<(unsigned)std::min<size_t>(1184, (cnt + 255) / 256), 256, 0, cs>>>(
                (const double*)(xs + (size_t)r0 * n * es), (int64_t)cnt, c->nf_flag.as<int32_t>());
            else dev::nonfinite_kernel<float><<<(unsigned)std::min<size_t>(1184, (cnt + 255) / 256), 256, 0, cs>>>(
                (const float*)(xs + (size_t)r0 * n * es), (int64_t)cnt, c->nf_flag.as<int32_t>());
            c->launches += 1;
        }
        eval_device(c, xs + (size_t)r0 * n * es, Bc, c->f_stage.as<double>() + r0, grad_out ? gs + (size_t)r0 * n * es : nullptr,
                    unsat_out ? c->u_stage.as<int32_t>() + r0 : nullptr, cs, false, dual && i == 1 ? &c->scr2 : nullptr);
        CK(cudaEventRecord(c->ev_done[(size_t)i], cs));
        CK(cudaStreamWaitEvent(c->copy_d2h, c->ev_done[(size_t)i], 0));
        const int64_t nr = r1 - r0;
        if (nr > 0) {
            CK(cudaMemcpyAsync(f_out + r0, c->f_stage.as<double>() + r0, (size_t)nr * 8, cudaMemcpyDeviceToHost, c->copy_d2h));
            if (grad_out && n) CK(cudaMemcpyAsync((char*)grad_out + (size_t)r0 * n * es, gs + (size_t)r0 * n * es, (size_t)nr * n * es,
                                                  cudaMemcpyDeviceToHost, c->copy_d2h));
            if (unsat_out) CK(cudaMemcpyAsync(unsat_out + r0, c->u_stage.as<int32_t>() + r0, (size_t)nr * 4, cudaMemcpyDeviceToHost, c->copy_d2h));
        }
    }
    CK(cudaMemcpyAsync(c->nf_host, c->nf_flag.p, 4, cudaMemcpyDeviceToHost, c->copy_d2h));
    CK(cudaStreamSynchronize(c->copy_d2h));
    if (dual) CK(cudaStreamSynchronize(c->comp2));
    CK(cudaStreamSynchronize(st));
    if (*c->nf_host) throw Error(FFSAT_ERR_NONFINITE, "non-finite point coordinate");
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_set_weights(ffsat_ctx* c, const double* w, int32_t on_device, void* stream) {
    ABI_TRY(c)
    need_device(c);
    if (!w) throw Error(FFSAT_ERR_ARG, "null weights");
    const int64_t m = c->Lo.m;
    if (m == 0) return FFSAT_OK;
    cudaStream_t st = S(stream);
    const double* src = w;
    if (!on_device) {
        for (int64_t i = 0; i < m; ++i) if (!std::isfinite(w[i])) throw Error(FFSAT_ERR_NONFINITE, "non-finite weight");
        c->w_stage.ensure((size_t)m * 8);
        CK(cudaMemcpyAsync(c->w_stage.p, w, (size_t)m * 8, cudaMemcpyHostToDevice, st));
        src = c->w_stage.as<double>();
    }
    if (c->Lo.precision == 64) dev::permute_weights_kernel<double><<<blocks_for(m, 256), 256, 0, st>>>(c->w_pos.as<double>(), src, c->order.as<int64_t>(), m);
    else dev::permute_weights_kernel<float><<<blocks_for(m, 256), 256, 0, st>>>(c->w_pos.as<float>(), src, c->order.as<int64_t>(), m);
    CK(cudaGetLastError());
    if (!on_device) CK(cudaStreamSynchronize(st));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_get_weights(ffsat_ctx* c, double* w, int32_t on_device, void* stream) {
    ABI_TRY(c)
    need_device(c);
    if (!w) throw Error(FFSAT_ERR_ARG, "null weights");
    const int64_t m = c->Lo.m;
    if (m == 0) return FFSAT_OK;
    cudaStream_t st = S(stream);
    double* dst = w;
    if (!on_device) {
        c->w_stage.ensure((size_t)m * 8);
        dst = c->w_stage.as<double>();
    }
    if (c->Lo.precision == 64) dev::unpermute_weights_kernel<double><<<blocks_for(m, 256), 256, 0, st>>>(dst, c->w_pos.as<double>(), c->order.as<int64_t>(), m);
    else dev::unpermute_weights_kernel<float><<<blocks_for(m, 256), 256, 0, st>>>(dst, c->w_pos.as<float>(), c->order.as<int64_t>(), m);
    CK(cudaGetLastError());
    if (!on_device) {
        CK(cudaMemcpyAsync(w, dst, (size_t)m * 8, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_check(const ffsat_ctx* c, const int8_t* a, int64_t* n_unsat, double* fw) {
    ABI_TRY(nullptr)
    if (!c || !a) throw Error(FFSAT_ERR_ARG, "null argument");
    for (int32_t v = 0; v < c->F.n; ++v)
        if (a[v] != 1 && a[v] != -1) throw Error(FFSAT_ERR_ARG, "assignment entries must be -1 or +1");
    int64_t cnt = exact_unsat(c->F, a, fw);
    if (n_unsat) *n_unsat = cnt;
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_search_create(ffsat_ctx* c, int64_t batch, int64_t point0, uint64_t seed, const ffsat_solve_params* params,
                                 ffsat_search** out) {
    ABI_TRY(c)
    need_device(c);
    if (!out || batch <= 0 || point0 < 0 || point0 + batch > (int64_t)UINT32_MAX) throw Error(FFSAT_ERR_ARG, "bad search arguments");
    *out = nullptr;
    std::unique_ptr<ffsat_search> s(new ffsat_search());
    s->ctx = c;
    s->B = batch;
    s->point0 = point0;
    s->seed = seed;
    ffsat_default_params(&s->P);
    if (params) s->P = *params;
    check_params(s->P);
    search_alloc(s.get());
    // the search's weights start from the formula's static weights (w0 = 1 for unweighted formulas, #15);
    // they are the search's own ERWA state: the context's weights (ffsat_set_weights) and other searches are untouched
    const int64_t m = c->Lo.m;
    if (m > 0) {
        if (c->Lo.precision == 64) dev::permute_weights_kernel<double><<<blocks_for(m, 256), 256>>>(s->W.as<double>(), c->w_static_orig.as<double>(), c->order.as<int64_t>(), m);
        else dev::permute_weights_kernel<float><<<blocks_for(m, 256), 256>>>(s->W.as<float>(), c->w_static_orig.as<double>(), c->order.as<int64_t>(), m);
    }
    const int64_t tot = batch * c->Lo.n;
    if (tot > 0) {
        if (c->Lo.precision == 64) dev::init_points_kernel<double><<<blocks_for(tot, 256), 256>>>(s->X.as<double>(), batch, c->Lo.n, seed, point0, 0);
        else dev::init_points_kernel<float><<<blocks_for(tot, 256), 256>>>(s->X.as<float>(), batch, c->Lo.n, seed, point0, 0);
    }
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    *out = s.release();
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_set_x(ffsat_search* s, const void* x, int32_t on_device, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s || !x) throw Error(FFSAT_ERR_ARG, "null argument");
    need_device(c);
    const size_t bytes = (size_t)s->B * c->Lo.n * c->esize;
    CK(cudaMemcpyAsync(s->X.p, x, bytes, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, S(stream)));
    if (!on_device) CK(cudaStreamSynchronize(S(stream)));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_begin_round(ffsat_search* s, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s) throw Error(FFSAT_ERR_ARG, "null search");
    need_device(c);
    search_begin_round(s, S(stream));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_iterate(ffsat_search* s, int32_t n_iters, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s || n_iters < 0) throw Error(FFSAT_ERR_ARG, "bad iterate arguments");
    need_device(c);
    search_iterate(s, n_iters, S(stream));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_check(ffsat_search* s, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s) throw Error(FFSAT_ERR_ARG, "null search");
    need_device(c);
    search_check(s, S(stream));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_restart(ffsat_search* s, const int32_t* U_global, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s) throw Error(FFSAT_ERR_ARG, "null search");
    need_device(c);
    search_restart(s, U_global, S(stream));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_reduce(ffsat_search* s, void* stream) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s) throw Error(FFSAT_ERR_ARG, "null search");
    need_device(c);
    search_reduce(s, S(stream));
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_stats_get(ffsat_search* s, void* stream, ffsat_search_stats* out) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s || !out) throw Error(FFSAT_ERR_ARG, "null argument");
    need_device(c);
    search_stats(s, S(stream), out);
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_get_buffers(ffsat_search* s, ffsat_search_buffers* o) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s || !o) throw Error(FFSAT_ERR_ARG, "null argument");
    o->x = s->X.p; o->grad = s->Gx.p; o->f = s->fX.as<double>(); o->eta = s->eta.as<double>();
    o->unsat = s->unsat.as<int32_t>(); o->U = s->U.as<int32_t>(); o->weights = s->W.p;
    o->keys = s->stats.as<int64_t>() + 1; o->solved = s->solved.as<int32_t>();
    o->xp = s->Xp.p;
    o->x_prev = s->Xm.p; o->y = s->Y.p; o->f_y = s->fy.as<double>(); o->t = s->tmom.as<double>();
    o->phase = s->phase.as<int32_t>();
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_search_assignment(ffsat_search* s, int64_t lp, int8_t* out) {
    ffsat_ctx* c = s ? s->ctx : nullptr;
    ABI_TRY(c)
    if (!s || !out || lp < 0 || lp >= s->B) throw Error(FFSAT_ERR_ARG, "bad assignment arguments");
    need_device(c);
    search_assignment(s, lp, out);
    return FFSAT_OK;
    ABI_CATCH(c)
}

void ffsat_search_free(ffsat_search* s) { delete s; }

ffsat_status ffsat_solve(ffsat_ctx* c, int64_t batch, int64_t max_restarts, uint64_t seed, const ffsat_solve_params* params,
                         int8_t* assignment_out, ffsat_result* res) {
    ABI_TRY(c)
    if (!assignment_out || !res || max_restarts < 1) throw Error(FFSAT_ERR_ARG, "bad solve arguments");
    need_device(c);
    auto t0 = std::chrono::steady_clock::now();
    ffsat_search* sp = nullptr;
    ffsat_status st0 = ffsat_search_create(c, batch, 0, seed, params, &sp);
    if (st0 != FFSAT_OK) return st0;
    std::unique_ptr<ffsat_search> s(sp);
    cudaStream_t st = nullptr;
    const int n = c->Lo.n;
    std::vector<int8_t> cand((size_t)n), best((size_t)n, 1);
    int64_t best_cnt = INT64_MAX;
    double best_w = 0;
    std::memset(res, 0, sizeof(*res));
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    auto consider = [&](int64_t lp) {
        search_assignment(s.get(), lp, cand.data());
        double fw = 0;
        int64_t cnt = exact_unsat(c->F, cand.data(), &fw);
        if (cnt < best_cnt || (cnt == best_cnt && fw < best_w)) {
            best_cnt = cnt;
            best_w = fw;
            best = cand;
        }
        return cnt == 0;
    };
    bool sat = false;
    const ffsat_solve_params& P = s->P;
    for (int64_t r = 0; r < max_restarts && !sat; ++r) {
        search_begin_round(s.get(), st);
        ffsat_search_stats ss{};
        int it = 0;
        while (it < P.max_inner) {
            int step = std::min(P.check_every, P.max_inner - it);
            search_iterate(s.get(), step, st);
            it += step;
            search_stats(s.get(), st, &ss);
            res->iterations += step;
            if (ss.solved_point >= 0 || ss.active == 0) break;
            if (P.timeout_s > 0 && elapsed() > P.timeout_s) break;
        }
        search_stats(s.get(), st, &ss);
        if (ss.solved_point >= 0 && consider(ss.solved_point)) sat = true;
        search_check(s.get(), st);
        search_stats(s.get(), st, &ss);
        res->restarts = r + 1;
        if (!sat && ss.best_point >= 0 && consider(ss.best_point)) sat = true;
        if (sat) break;
        if (P.timeout_s > 0 && elapsed() > P.timeout_s) break;
        search_restart(s.get(), nullptr, st);
    }
    CK(cudaStreamSynchronize(st));
    std::memcpy(assignment_out, best.data(), (size_t)n);
    res->sat = sat ? 1 : 0;
    res->best_unsat = best_cnt == INT64_MAX ? -1 : best_cnt;
    res->best_falsified_weight = best_w;
    res->seconds = elapsed();
    return FFSAT_OK;
    ABI_CATCH(c)
}

ffsat_status ffsat_layout_units(const ffsat_ctx* c, int64_t* n_units, int64_t* units_out, int64_t cap, int64_t* order_out) {
    ABI_TRY(nullptr)
    if (!c || !n_units) throw Error(FFSAT_ERR_ARG, "null argument");
    const Layout& L = c->Lo;
    *n_units = (int64_t)L.units.size();
    if (units_out)
        for (int64_t u = 0; u < std::min<int64_t>(cap, (int64_t)L.units.size()); ++u) {
            const WorkUnit& w = L.units[(size_t)u];
            units_out[4 * u] = w.bucket;
            units_out[4 * u + 1] = w.count;
            units_out[4 * u + 2] = w.pos_begin;
            units_out[4 * u + 3] = L.path == 1 ? 1 : 0;
        }
    if (order_out) std::copy(L.order.begin(), L.order.end(), order_out);
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_launch_count(const ffsat_ctx* c, int64_t* out) {
    ABI_TRY(nullptr)
    if (!c || !out) throw Error(FFSAT_ERR_ARG, "null argument");
    *out = c->launches;
    return FFSAT_OK;
    ABI_CATCH(nullptr)
}

ffsat_status ffsat_eval_profiled(ffsat_ctx* c, const void* x, int64_t B, double* f_out, void* grad_out, int32_t* unsat_out,
                                 void* stream, double* ms4) {
    ABI_TRY(c)
    need_device(c);
    if (B <= 0 || !x || !f_out || !ms4) throw Error(FFSAT_ERR_ARG, "bad profiled eval arguments");
    for (cudaEvent_t& e : c->ev)
        if (!e) CK(cudaEventCreate(&e));
    cudaStream_t st = S(stream);
    eval_device(c, x, B, f_out, grad_out, unsat_out, st, true);
    CK(cudaEventSynchronize(c->ev[4]));
    for (int i = 0; i < 4; ++i) {
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]));
        ms4[i] = ms;
    }
    return FFSAT_OK;
    ABI_CATCH(c)
}

void ffsat_free(ffsat_ctx* c) { delete c; }

}  // extern "C"
