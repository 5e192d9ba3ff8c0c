/*
 * oracle/dp.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 CPU oracle (tier T2) for the objective
 *     f(x) = sum_c w_c * FE_c(x)                      (Def. 3, Eq. 5)
 * and its gradient, for formulas of symmetric constraints.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may load
 * this file's shared object.  It shares no code, header, table or constant
 * generator with the CUDA product path (paper_2308_15020_b200/csrc).
 *
 * FE_c is the Walsh expansion of constraint c (Thm. 1): the unique
 * multilinear polynomial equal to the +-1 truth value (-1 = True) at every
 * corner.  For a symmetric constraint it is evaluated here exactly as GradSAT's
 * belief propagation on the constraint's BDD (Alg. 5, Eg. 5/6): the
 * BDD of a symmetric constraint has one node per (literal position i, number t
 * of True literals among the first i), so
 *   M_TD  (top-down)  = q_i(t): probability that t of the first i
 *          literals are True under randomized rounding P[l = True] = (1-l)/2;
 *   M_BU  (bottom-up) = beta_i(t): expected truth value f(T) given
 *          t Trues among the first i literals; beta_k(t) = f(t).
 *   FE    = beta_0(0) = sum_t f(t) q_k(t)        (Eg. 5: FE = P(false) - P(true))
 *   dFE/dl_i = 1/2 * sum_t q_{i-1}(t) (beta_i(t) - beta_i(t+1))
 *          which is P:791's M_TD[v](M_BU[v.true] - M_BU[v.false]) written with
 *          beta = 1 - 2*P(sat) (reading #8 of DESIGN.md, reproduces Eg. 6's 19/64, 33/64).
 * Literal values are l = s*x_v with s = -1 for a negated literal.  The chain
 * rule (Prop. 1) gives d f / d x_v = sum over occurrences of
 * w_c * s * dFE/dl_i.  f and grad are summed in fp64 in ascending constraint,
 * then literal-position, order.
 *
 * Discrete check (Thm. 4; Alg. 1 line 5): variable v is True
 * iff x_v < 0 (x = 0 and -0.0 are False, reading #10); a constraint
 * is satisfied iff its count t of True literals satisfies its kind.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_ = 0, XOR_ = 1, XNOR_ = 2, CARD_GE_ = 3, CARD_LE_ = 4, NAE_ = 5 };

/* Constraint semantics by count t of True literals among k. */
static int sat_by_count(int kind, int k, int bound, int t) {
    switch (kind) {
    case OR_: return t >= 1;
    case XOR_: return (t & 1) == 1;     /* odd parity */
    case XNOR_: return (t & 1) == 0;    /* even parity */
    case CARD_GE_: return t >= bound;   /* at least `bound` True literals (Eg. 1) */
    case CARD_LE_: return t <= bound;   /* at most `bound` True literals */
    case NAE_: return t > 0 && t < k;   /* not all equal */
    default: return 0;
    }
}

/* One constraint by the BDD/probability DP.  l[k] literal values, dl[k] output (may be NULL).
 * q must hold (k+1)(k+2)/2 doubles (triangular rows q_i(0..i)), b0,b1 k+2 doubles each. */
static double constraint_dp(int kind, int k, int bound, const double* l, double* dl,
                            double* q, double* b0, double* b1) {
    /* forward (top-down messages) */
    q[0] = 1.0;
    size_t row = 0; /* offset of row i-1 */
    for (int i = 1; i <= k; ++i) {
        double p = (1.0 - l[i - 1]) * 0.5; /* P[literal i True] */
        const double* prev = q + row;
        double* cur = q + row + (size_t)i;   /* row i starts after row i-1 (length i) */
        for (int t = 0; t <= i; ++t) {
            double stay = (t <= i - 1) ? prev[t] : 0.0;
            double up = (t >= 1) ? prev[t - 1] : 0.0;
            cur[t] = (1.0 - p) * stay + p * up;
        }
        row += (size_t)i;
    }
    /* row k offset = k(k+1)/2 */
    const double* qk = q + (size_t)k * (size_t)(k + 1) / 2;
    double fe = 0.0;
    for (int t = 0; t <= k; ++t) fe += (sat_by_count(kind, k, bound, t) ? -1.0 : 1.0) * qk[t];
    if (!dl) return fe;
    /* backward (bottom-up messages) */
    double* bi = b0; double* bn = b1;
    for (int t = 0; t <= k; ++t) bi[t] = sat_by_count(kind, k, bound, t) ? -1.0 : 1.0;
    for (int i = k; i >= 1; --i) {
        const double* qp = q + (size_t)(i - 1) * (size_t)i / 2; /* row i-1 */
        double s = 0.0;
        for (int t = 0; t <= i - 1; ++t) s += qp[t] * (bi[t] - bi[t + 1]);
        dl[i - 1] = 0.5 * s;
        double p = (1.0 - l[i - 1]) * 0.5;
        for (int t = 0; t <= i - 1; ++t) bn[t] = (1.0 - p) * bi[t] + p * bi[t + 1];
        double* tmp = bi; bi = bn; bn = tmp;
    }
    return fe;
}

/* Single constraint entry point (tests): returns FE, writes dFE/dl_i into dl (nullable). */
double oracle_constraint(int kind, int k, int bound, const double* l, double* dl) {
    double* q = (double*)malloc(sizeof(double) * ((size_t)(k + 1) * (size_t)(k + 2) / 2 + 1));
    double* b0 = (double*)malloc(sizeof(double) * (size_t)(k + 2));
    double* b1 = (double*)malloc(sizeof(double) * (size_t)(k + 2));
    double fe = constraint_dp(kind, k, bound, l, dl, q, b0, b1);
    free(q); free(b0); free(b1);
    return fe;
}

/* BDD messages of one constraint (Eg. 5/6 pins): q_tri and beta_tri are triangular tables with
 * row i (i = 0..k) of length i+1 at offset i(i+1)/2; q = M_TD (probability of t Trues among the
 * first i literals), beta = expected truth value given t Trues among the first i (M_BU in the
 * +-1 encoding: P(sat | node) = (1 - beta)/2). */
void oracle_messages(int kind, int k, int bound, const double* l, double* q_tri, double* beta_tri) {
    double* b0 = (double*)malloc(sizeof(double) * (size_t)(k + 2));
    double* b1 = (double*)malloc(sizeof(double) * (size_t)(k + 2));
    double* dl = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    constraint_dp(kind, k, bound, l, dl, q_tri, b0, b1);
    /* re-run the backward recursion keeping every row */
    double* row = beta_tri + (size_t)k * (size_t)(k + 1) / 2;
    for (int t = 0; t <= k; ++t) row[t] = sat_by_count(kind, k, bound, t) ? -1.0 : 1.0;
    for (int i = k; i >= 1; --i) {
        const double* bi = beta_tri + (size_t)i * (size_t)(i + 1) / 2;
        double* bp = beta_tri + (size_t)(i - 1) * (size_t)i / 2;
        double p = (1.0 - l[i - 1]) * 0.5;
        for (int t = 0; t <= i - 1; ++t) bp[t] = (1.0 - p) * bi[t] + p * bi[t + 1];
    }
    free(b0); free(b1); free(dl);
}

/* f[b] and grad[b][n] for B points x[b][n] (row-major).  lits are DIMACS (1-based, sign = polarity).
 * weight NULL means all 1.  grad may be NULL.  Returns 0. */
int oracle_eval(int32_t n, int64_t m, const uint8_t* kind, const int32_t* bound, const double* weight,
                const int64_t* offsets, const int32_t* lits, int64_t B, const double* x, double* f,
                double* grad, int nthreads) {
    int kmax = 0;
    for (int64_t c = 0; c < m; ++c) {
        int k = (int)(offsets[c + 1] - offsets[c]);
        if (k > kmax) kmax = k;
    }
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        double* q = (double*)malloc(sizeof(double) * ((size_t)(kmax + 1) * (size_t)(kmax + 2) / 2 + 1));
        double* b0 = (double*)malloc(sizeof(double) * (size_t)(kmax + 2));
        double* b1 = (double*)malloc(sizeof(double) * (size_t)(kmax + 2));
        double* l = (double*)malloc(sizeof(double) * (size_t)(kmax + 1));
        double* dl = (double*)malloc(sizeof(double) * (size_t)(kmax + 1));
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t b = 0; b < B; ++b) {
            const double* xb = x + b * (int64_t)n;
            double* gb = grad ? grad + b * (int64_t)n : NULL;
            if (gb) memset(gb, 0, sizeof(double) * (size_t)n);
            double fb = 0.0;
            for (int64_t c = 0; c < m; ++c) {
                int k = (int)(offsets[c + 1] - offsets[c]);
                const int32_t* lc = lits + offsets[c];
                for (int i = 0; i < k; ++i) {
                    int32_t lit = lc[i];
                    int32_t v = lit > 0 ? lit - 1 : -lit - 1;
                    l[i] = lit > 0 ? xb[v] : -xb[v];
                }
                double w = weight ? weight[c] : 1.0;
                double fe = constraint_dp(kind[c], k, bound ? bound[c] : 0, l, gb ? dl : NULL, q, b0, b1);
                fb += w * fe;
                if (gb) {
                    for (int i = 0; i < k; ++i) {
                        int32_t lit = lc[i];
                        int32_t v = lit > 0 ? lit - 1 : -lit - 1;
                        gb[v] += w * (lit > 0 ? dl[i] : -dl[i]);
                    }
                }
            }
            f[b] = fb;
        }
        free(q); free(b0); free(b1); free(l); free(dl);
    }
    return 0;
}

/* Discrete check of sgn(x) for B points: n_unsat[b], falsified_weight[b] (nullable) and
 * U[c] = number of points whose rounded assignment leaves c unsatisfied (nullable). */
int oracle_check(int32_t n, int64_t m, const uint8_t* kind, const int32_t* bound, const double* weight,
                 const int64_t* offsets, const int32_t* lits, int64_t B, const double* x,
                 int64_t* n_unsat, double* falsified_weight, int32_t* U) {
    if (U) memset(U, 0, sizeof(int32_t) * (size_t)m);
    for (int64_t b = 0; b < B; ++b) {
        const double* xb = x + b * (int64_t)n;
        int64_t cnt = 0;
        double fw = 0.0;
        for (int64_t c = 0; c < m; ++c) {
            int k = (int)(offsets[c + 1] - offsets[c]);
            int t = 0;
            for (int i = 0; i < k; ++i) {
                int32_t lit = lits[offsets[c] + i];
                int32_t v = lit > 0 ? lit - 1 : -lit - 1;
                int var_true = xb[v] < 0.0;
                int lit_true = lit > 0 ? var_true : !var_true;
                t += lit_true;
            }
            if (!sat_by_count(kind[c], k, bound ? bound[c] : 0, t)) {
                ++cnt;
                fw += weight ? weight[c] : 1.0;
                if (U) ++U[c];
            }
        }
        if (n_unsat) n_unsat[b] = cnt;
        if (falsified_weight) falsified_weight[b] = fw;
    }
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
