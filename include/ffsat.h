/*
 * ffsat.h -- C-ABI of libffsat.so, the B200-native FastFourierSAT hot path.
 *
 * What it computes (PAPER.md = arXiv 2308.15020, cited as P:<line>):
 *   f(x)  = sum_c w_c * FE_c(x)        objective, Def. 3 / Eq. 5
 *   FE_c  = Walsh expansion of the symmetric constraint c (Thm. 1), -1 = True,
 *           evaluated by the product-at-roots-of-unity view of Alg. 2 / Eqs. 6-9
 *   grad f by reverse differentiation of that product (Prop. 1, Eq. 10)
 *   the CLS loop of Alg. 1: projected gradient descent (Alg. 4),
 *   sign rounding + exact constraint check (Thm. 4), ERWA weights (Prop. 3,
 *   P:584-605) and O/F/R rephasing.
 * DESIGN.md lists every reading taken where the paper is silent or garbled.
 *
 * Conventions for every entry point:
 *   - Every call returns an ffsat_status and never aborts; C++ exceptions never cross this ABI.
 *     On failure ffsat_last_error(ctx) (or ffsat_last_error(NULL) before a context exists,
 *     thread-local) returns a message (parse errors carry the 1-based line number).
 *   - The caller owns every buffer it passes.  ffsat_load* deep-copy the formula: the caller may
 *     free its arrays after the call returns.
 *   - "on_device = 1": every buffer argument of that call is a device pointer on the context's
 *     device and work is enqueued on `stream` (a cudaStream_t, NULL = legacy default stream);
 *     the call returns without synchronising.  "on_device = 0": buffers are host memory; the
 *     library stages them through its own device buffers and synchronises `stream` before return.
 *   - Points are row-major [B][n] in the context dtype (float if precision 32, double if 64).
 *   - A context is not thread-safe: one context per host thread, or external synchronisation.
 *   - There is no CPU fallback: a context needs a CUDA device (except device = -1 host-only
 *     contexts, which parse/validate/check but refuse every compute call with FFSAT_ERR_ARG).
 */
#ifndef FFSAT_H
#define FFSAT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFSAT_ABI_VERSION 1

typedef struct ffsat_ctx ffsat_ctx;       /* opaque: formula, device layout, weights */
typedef struct ffsat_search ffsat_search; /* opaque: device-resident batched CLS state */

typedef enum {
    FFSAT_OK = 0,
    FFSAT_ERR_ARG = 1,        /* bad argument / unsupported configuration */
    FFSAT_ERR_PARSE = 2,      /* text syntax error (message has the line number) */
    FFSAT_ERR_RANGE = 3,      /* literal variable outside [1, n_vars] */
    FFSAT_ERR_DUPVAR = 4,     /* a variable appears twice in one constraint (#13) */
    FFSAT_ERR_BOUND = 5,      /* cardinality bound outside [0, k] (#14) */
    FFSAT_ERR_NONFINITE = 6,  /* NaN/Inf weight or point coordinate */
    FFSAT_ERR_CUDA = 7,       /* CUDA runtime failure (including "no device") */
    FFSAT_ERR_NCCL = 8,       /* reserved: collectives run in the caller (torch.distributed) */
    FFSAT_ERR_OOM = 9         /* device allocation failed */
} ffsat_status;

/* Constraint kinds (at-most and NAE are this build's extension, #12).
 * t = number of True literals of the constraint. */
typedef enum {
    FFSAT_OR = 0,       /* t >= 1                         (CNF clause)          */
    FFSAT_XOR = 1,      /* t odd                          (App. B)   */
    FFSAT_XNOR = 2,     /* t even                                               */
    FFSAT_CARD_GE = 3,  /* t >= bound   (Eg. 1 reading, #11)           */
    FFSAT_CARD_LE = 4,  /* t <= bound                                           */
    FFSAT_NAE = 5       /* 0 < t < k                                            */
} ffsat_kind;

/* A formula as arrays (Alg. 1 input).  lits are DIMACS literals (1-based variable index,
 * negative = negated).  Constraint c owns lits[offsets[c] .. offsets[c+1]).  bound is read for
 * CARD_GE / CARD_LE only (NULL = all 0).  weight NULL = all 1 (static weights w_c, Def. 3). */
typedef struct {
    int32_t n_vars;
    int64_t n_cons;
    const uint8_t* kind;     /* [n_cons] ffsat_kind */
    const int32_t* bound;    /* [n_cons] or NULL */
    const double* weight;    /* [n_cons] or NULL */
    const int64_t* offsets;  /* [n_cons + 1], offsets[0] = 0, non-decreasing */
    const int32_t* lits;     /* [offsets[n_cons]] */
} ffsat_formula;

typedef struct {
    int32_t precision;  /* 0 = auto (64 iff some non-fast-path constraint has k > 64), 32, 64 */
    int32_t device;     /* CUDA device ordinal; -1 = host-only context (no GPU needed) */
    int32_t path;       /* 0 = auto, 1 = force on-chip tiled fast path (64-point kernel when eligible, its TMEM
                           variant when n <= 256), 2 = force global path, 3 = tiled path with the 32-point kernel
                           only, 4 = tiled path without the TMEM variant (64-point shared-memory kernel) */
    int32_t batch_ref;  /* reference batch of the launch plan, 0 = 1024.  The fast kernels' split of the
                           constraints into chunks (and so every partial sum) is planned once, at load, for
                           this batch size and reused for every call: a point's f / grad / unsat bits do not
                           depend on the batch it is evaluated in (restart sharding over any number of GPUs
                           reproduces the single-GPU trajectories, F7).  Set it to the batch you
                           evaluate for best throughput (a much smaller batch than batch_ref underfills the GPU). */
} ffsat_options;

typedef struct {
    int32_t n_vars;
    int32_t precision;      /* 32 or 64 */
    int64_t n_cons;
    int64_t n_lits;         /* sum_c k_c: literal-gradient terms per point */
    int64_t n_fast_cons;    /* constraints on the product fast paths (OR/AND/NAE/XOR-type, F3) */
    int64_t n_sym_cons;     /* constraints on the root-of-unity product path */
    int64_t n_fast_lits;
    int64_t n_sym_lits;
    int64_t sym_root_lits;  /* sum over root-of-unity-path sym constraints of k * M', M' = floor((k+1)/2) */
    int32_t path;           /* 1 tiled, 2 global */
    int32_t wide;           /* tiled path kernel: 0 = 32-point, 1 = 64-point (two points per lane) with the gradient tile
                               in shared memory, 2 = 64-point with the gradient tile in tensor memory (TMEM) */
    int32_t max_k;
    int64_t device_bytes;   /* persistent device memory held by the context */
    int64_t n_own_lits;     /* global path: literals of the short constraints whose gradient terms the owner-computes
                               kernel forms per variable (no T-buffer round trip; SURVEY 8(e) "owner-computes").  On
                               by default when the fast constraints are one bucket of k <= 3 clauses (uniform random
                               3-SAT, c5); environment FFSAT_OWN=0 disables it, FFSAT_OWN=1 extends it to every
                               k <= 3 bucket.  Results agree within the stated tolerance either way (the summation
                               order differs); 0 when not used */
    int64_t n_tree_cons;    /* fp64 symmetric constraints on the product-tree path (long k) */
    int64_t tree_work;      /* their FP64 instructions per point (the tree path's algorithmic count) */
} ffsat_info_t;

/* Build a context from arrays (validates, buckets, precomputes coefficients, uploads). */
ffsat_status ffsat_load(const ffsat_formula* formula, const ffsat_options* opt, ffsat_ctx** out);
/* Same from a text file: "p cnf", "p hnf", "p whnf" (SPEC S:99-104 grammar) plus this build's
 * `a <b> <lits> 0` (at most b) and `n <lits> 0` (NAE).  Parse errors report the line. */
ffsat_status ffsat_load_file(const char* path, const ffsat_options* opt, ffsat_ctx** out);
ffsat_status ffsat_info(const ffsat_ctx* ctx, ffsat_info_t* out);
/* Copy the parsed formula back out (host arrays sized from ffsat_info; any pointer may be NULL). */
ffsat_status ffsat_export(const ffsat_ctx* ctx, uint8_t* kind, int32_t* bound, double* weight,
                          int64_t* offsets, int32_t* lits);

/* f[b] = sum_c w_c FE_c(x_b) (fp64 accumulation), grad[b][:] = d f / d x at x_b (context dtype),
 * unsat[b] = number of constraints falsified by sgn(x_b) (x < 0 = True, x = 0 = False; exact).
 * x: [B][n] context dtype, coordinates in [-1, 1] (not checked on device; host inputs are
 * checked for NaN/Inf -> FFSAT_ERR_NONFINITE, detected by a device kernel on the staged copy: the
 * outputs are then unspecified).  f_out [B] double; grad_out [B][n] or NULL; unsat_out [B] int32 or
 * NULL.  Weights: the context's current weights (ffsat_set_weights).
 * Host buffers (on_device = 0) are staged in up to 4 equal chunks of at least batch_ref points whose H2D / D2H copies overlap
 * the chunk evaluations; pinned host memory is needed for the overlap (pageable memory still works).
 * The call returns when the outputs are in host memory.  Device buffers (on_device = 1) are asynchronous
 * on `stream`.  B = 0 is a no-op.  Results per point do not depend on B or on the point's position in the
 * batch (the launch plan is batch-independent, ffsat_options.batch_ref): host and device buffers give the same
 * bits. */
ffsat_status ffsat_eval(ffsat_ctx* ctx, const void* x, int64_t B, int32_t on_device, double* f_out,
                        void* grad_out, int32_t* unsat_out, void* stream);

/* Current weights w_c (constraint order of the input formula), double [n_cons]. */
ffsat_status ffsat_set_weights(ffsat_ctx* ctx, const double* w, int32_t on_device, void* stream);
ffsat_status ffsat_get_weights(ffsat_ctx* ctx, double* w, int32_t on_device, void* stream);

/* Exact check of one assignment (host, int8 [n]: -1 = True, +1 = False, Alg. 1 output P:219):
 * number of falsified constraints and their total static weight (Thm. 4 realised discretely). */
ffsat_status ffsat_check(const ffsat_ctx* ctx, const int8_t* assignment, int64_t* n_unsat,
                         double* falsified_weight);

/* ---- batched CLS search state (Alg. 1 with p_t = batch points; restart sharding uses point0) ---- */
typedef struct {
    double eta0;             /* initial / maximal step (default 1.0) */
    double eta_min;          /* stop when eta < eta_min (default 1e-12) */
    double armijo_c1;        /* sufficient-decrease constant (default 1e-4) */
    double alpha;            /* ERWA decay (default 0.4) */
    int32_t max_inner;       /* PGD trials per restart round (default 500) */
    int32_t check_every;     /* every check_every-th PGD iteration of a round evaluates the trial points with the
                                fused exact check of their rounded assignment (A9; a satisfying trial is captured
                                as solved); the others skip it.  ffsat_solve polls after those iterations (default 10) */
    int32_t policy;          /* rephasing cycle: 0 = ROF, 1 = RF, 2 = R */
    int32_t adaptive_weights;/* 1 = ERWA (decision mode), 0 = fixed weights */
    double timeout_s;        /* ffsat_solve wall-clock limit, <= 0 = none */
    int32_t accel;           /* 0 = monotone projected Armijo backtracking, one trial per iteration (#16);
                                1 = FISTA: accelerated projected gradient with backtracking on the quadratic upper
                                bound ("FISTA", #16b), one evaluation (trial or extrapolation point)
                                per iteration.  In this mode ffsat_search_buffers.grad holds the gradient at the
                                extrapolation point y, f and x the last accepted iterate (default 0) */
    int32_t reserved;        /* must be 0 */
} ffsat_solve_params;

typedef struct {
    int64_t round;           /* restart rounds completed */
    int64_t iterations;      /* PGD iterations issued in the current round */
    int64_t active;          /* points not yet converged in the current round */
    int64_t solved_point;    /* lowest global point index whose trial or checked sgn(x) satisfied every constraint, -1 none */
    int64_t best_unsat;      /* minimum falsified count over points at the last check */
    int64_t best_point;      /* global index achieving best_unsat */
} ffsat_search_stats;

/* Device pointers owned by the search (for collectives and tests).  Per-constraint arrays (U, weights) are in the
 * library's POSITION order, not the input order of the formula: position p holds input constraint order[p], where
 * order is the map ffsat_layout_units returns (a permutation of 0..n_cons-1).  ffsat_search_restart expects a
 * U_global in the same position order (e.g. the element-wise SUM of every rank's U: all ranks share one layout). */
typedef struct {
    void* x;                 /* [B][n] accepted points */
    void* grad;              /* [B][n] gradient at x */
    double* f;               /* [B] f at x */
    double* eta;             /* [B] */
    int32_t* unsat;          /* [B] falsified count of sgn(x) at the last check */
    int32_t* U;              /* [n_cons] per-constraint falsified count over this batch at the last check (position order) */
    void* weights;           /* [n_cons] this search's current weights (context dtype, position order) */
    int64_t* keys;           /* [2] written by ffsat_search_reduce, MIN-reducible across ranks as they stand:
                                keys[0] = lowest GLOBAL point index whose solved flag is set, INT64_MAX if none;
                                keys[1] = (falsified count of sgn(x) at the last check << 32) | global point, minimised */
    int32_t* solved;         /* [B] 1 once a trial point or a checked point's sgn(x) satisfied every constraint */
    void* xp;                /* [B][n] the next point to evaluate (the trial; in FISTA mode possibly the point y) */
    /* FISTA state (params.accel = 1; NULL otherwise): */
    void* x_prev;            /* [B][n] x_{k-1} */
    void* y;                 /* [B][n] the extrapolation point whose gradient is in grad */
    double* f_y;             /* [B] f(y) */
    double* t;               /* [B] momentum t_k */
    int32_t* phase;          /* [B] 1: xp is a trial from y; 0: xp is the next y */
} ffsat_search_buffers;

ffsat_status ffsat_search_create(ffsat_ctx* ctx, int64_t batch, int64_t point0, uint64_t seed,
                                 const ffsat_solve_params* params, ffsat_search** out);
/* Overwrite the batch's points (device or host [B][n]) and restart the round at them. */
ffsat_status ffsat_search_set_x(ffsat_search* s, const void* x, int32_t on_device, void* stream);
/* Start a round: f, grad at the current x; eta = eta0; first trial point. */
ffsat_status ffsat_search_begin_round(ffsat_search* s, void* stream);
/* n PGD iterations (one batched f + grad evaluation each), enqueued on stream. */
ffsat_status ffsat_search_iterate(ffsat_search* s, int32_t n_iters, void* stream);
/* Check sgn(x) of every point: unsat[b], U[c] (over this batch, position order) on device; a point with unsat 0 is
 * marked solved and its assignment kept (ffsat_search_assignment), so a later restart cannot lose it. */
ffsat_status ffsat_search_check(ffsat_search* s, void* stream);
/* Reduce this batch's state into the device keys of ffsat_search_buffers (asynchronous on stream): the any-solved
 * key and the incumbent key, both in global point indices (point0 + local index).  Restart sharding MIN-all-reduces
 * them over ranks (C1, C4 of DESIGN.md section 6) without any host round trip. */
ffsat_status ffsat_search_reduce(ffsat_search* s, void* stream);
/* End the round: ERWA update of this search's weights with U_global (device int32 [n_cons], POSITION order; NULL =
 * this batch's U) when adaptive, then rephase every point (policy offset = global point index, #20). */
ffsat_status ffsat_search_restart(ffsat_search* s, const int32_t* U_global, void* stream);
/* ffsat_search_reduce + a synchronous read: solved_point / best_point are global point indices. */
ffsat_status ffsat_search_stats_get(ffsat_search* s, void* stream, ffsat_search_stats* out);
ffsat_status ffsat_search_get_buffers(ffsat_search* s, ffsat_search_buffers* out);
/* Assignment (-1 True / +1 False) of a local point: the solved trial assignment if that point
 * solved, else sgn of its current x. */
ffsat_status ffsat_search_assignment(ffsat_search* s, int64_t local_point, int8_t* assignment_out);
void ffsat_search_free(ffsat_search* s);

/* ---- single-GPU solve: Alg. 1 with p_t = batch ---- */
typedef struct {
    int32_t sat;                    /* 1 only with an assignment whose exact ffsat_check count is 0 */
    int32_t reserved;
    int64_t restarts;               /* rounds run */
    int64_t iterations;             /* PGD iterations run (each = one batched f + grad) */
    int64_t best_unsat;             /* exact falsified count of the returned assignment */
    double best_falsified_weight;   /* its falsified static weight */
    double seconds;
} ffsat_result;

ffsat_status ffsat_solve(ffsat_ctx* ctx, int64_t batch, int64_t max_restarts, uint64_t seed,
                         const ffsat_solve_params* params, int8_t* assignment_out /* [n] */,
                         ffsat_result* result);

void ffsat_default_params(ffsat_solve_params* p);

/* ---- diagnostics (used by bench.py) ---- */
/* Number of kernels this context has launched so far (every entry point). */
ffsat_status ffsat_launch_count(const ffsat_ctx* ctx, int64_t* out);
/* ffsat_eval on device buffers with CUDA events recorded on `stream` around each phase; synchronises
 * and writes the phase durations in ms: ms[0] fast-path product kernel (incl. transpose on the global
 * path), ms[1] root-path kernels, ms[2] gradient reduction, ms[3] f / unsat reduction. */
ffsat_status ffsat_eval_profiled(ffsat_ctx* ctx, const void* x, int64_t B, double* f_out, void* grad_out,
                                 int32_t* unsat_out, void* stream, double* ms4);
/* Layout introspection (tests; works on host-only contexts): the fast-path work units as rows
 * {bucket, count, first position, tiled (1) / global (0)} and the position -> input-constraint order.  With
 * units_out NULL only *n_units is written; otherwise cap rows at most are copied.  order_out: [n_cons] or NULL.
 * On the tiled path every unit is a var-disjoint class: no variable occurs in two of its constraints. */
ffsat_status ffsat_layout_units(const ffsat_ctx* ctx, int64_t* n_units, int64_t* units_out, int64_t cap,
                                int64_t* order_out);
const char* ffsat_last_error(const ffsat_ctx* ctx);
const char* ffsat_version(void);
void ffsat_free(ffsat_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FFSAT_H */
