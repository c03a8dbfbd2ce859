/*
 * axb_oracle.c — CPU ORACLE (test infrastructure only; see axb_oracle.h).
 *
 * Plain-C restatement of the reference engine, function by function, each
 * citing the reference file:line it follows (paths relative to
 * /root/reference/proj/include/axb/).  Build with -O2 -ffp-contract=off: the
 * reference's x86-64 build has no FMA, and the loops below keep its summation
 * order, so results are bitwise those of axb::Solver.
 */
#define _POSIX_C_SOURCE 200809L
#include "axb_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------------ */
/* RngStream — rng.hpp:18-123                                                */

static uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); } /* rng.hpp:107 */

static uint64_t mix_pure(uint64_t z) { /* rng.hpp:113-117 */
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

void orc_rng_init(orc_rng* r, uint64_t seed) { /* rng.hpp:20-25 */
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9e3779b97f4a7c15ULL; /* mix(): rng.hpp:109-112 */
        r->s[i] = mix_pure(x);
    }
    if (r->s[0] == 0 && r->s[1] == 0 && r->s[2] == 0 && r->s[3] == 0) r->s[0] = 1;
    r->seed = seed;
    r->spare = 0.0;
    r->has_spare = 0;
}

uint64_t orc_rng_next_u64(orc_rng* r) { /* rng.hpp:30-40, xoshiro256** */
    uint64_t* s = r->s;
    const uint64_t result = rotl64(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl64(s[3], 45);
    return result;
}

double orc_rng_next_unit(orc_rng* r) { /* rng.hpp:43 */
    return (double)(orc_rng_next_u64(r) >> 11) * 0x1.0p-53;
}

double orc_rng_gauss(orc_rng* r) { /* rng.hpp:46-59, Box–Muller with cached spare */
    if (r->has_spare) {
        r->has_spare = 0;
        return r->spare;
    }
    double u1 = ((double)(orc_rng_next_u64(r) >> 11) + 1.0) * 0x1.0p-53;
    double u2 = orc_rng_next_unit(r);
    double rad = sqrt(-2.0 * log(u1));
    double a = 2.0 * 3.141592653589793115997963468544185161590576171875 * u2; /* std::numbers::pi */
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}

void orc_rng_substream(const orc_rng* r, uint64_t t, orc_rng* out) { /* rng.hpp:102-104 */
    orc_rng_init(out, r->seed ^ mix_pure(0x5851f42d4c957f2dULL + t));
}

size_t orc_rng_categorical_cdf(orc_rng* r, const double* cum, size_t n, int* status) {
    /* rng.hpp:84-99: inverse transform + upper_bound, walk back over zero weights */
    double total = cum[n - 1];
    if (!(total > 0.0)) {
        if (status) *status = ORC_DOMAIN_ERROR;
        return 0;
    }
    double target = orc_rng_next_unit(r) * total;
    size_t lo = 0, hi = n - 1;
    while (lo < hi) {
        size_t mid = (lo + hi) / 2;
        if (cum[mid] <= target)
            lo = mid + 1;
        else
            hi = mid;
    }
    while (lo > 0 && cum[lo] == cum[lo - 1]) --lo;
    if (status) *status = ORC_OK;
    return lo;
}

void orc_dense_gaussian(orc_rng* r, size_t rows, size_t cols, double* out) { /* rng.hpp:126-131 */
    for (size_t i = 0; i < rows * cols; ++i) out[i] = orc_rng_gauss(r);
}

/* ------------------------------------------------------------------------ */
/* matrix.hpp primitives                                                     */

void orc_matmul(const double* a, size_t ar, size_t ac, const double* b, size_t bc, double* c) {
    /* matrix.hpp:325-338: ikj order, exact-zero a_ik skipped */
    memset(c, 0, sizeof(double) * ar * bc);
    for (size_t i = 0; i < ar; ++i) {
        double* ci = c + i * bc;
        for (size_t k = 0; k < ac; ++k) {
            double v = a[i * ac + k];
            if (v == 0.0) continue;
            const double* bk = b + k * bc;
            for (size_t j = 0; j < bc; ++j) ci[j] += v * bk[j];
        }
    }
}

void orc_gram_mmt(const double* a, size_t rows, size_t cols, double* g) { /* matrix.hpp:481-494 */
    for (size_t i = 0; i < rows; ++i) {
        const double* ri = a + i * cols;
        for (size_t j = i; j < rows; ++j) {
            const double* rj = a + j * cols;
            double s = 0.0;
            for (size_t k = 0; k < cols; ++k) s += ri[k] * rj[k];
            g[i * rows + j] = s;
            g[j * rows + i] = s;
        }
    }
}

double orc_frobenius_sq(const double* a, size_t len) { /* matrix.hpp:276-280 */
    double s = 0.0;
    for (size_t i = 0; i < len; ++i) s += a[i] * a[i];
    return s;
}

static void matvec(const double* m, size_t rows, size_t cols, const double* x, double* y) {
    /* matrix.hpp:400-410 */
    for (size_t i = 0; i < rows; ++i) {
        const double* ri = m + i * cols;
        double s = 0.0;
        for (size_t j = 0; j < cols; ++j) s += ri[j] * x[j];
        y[i] = s;
    }
}

static void matvec_transposed(const double* m, size_t rows, size_t cols, const double* x,
                              double* y) { /* matrix.hpp:420-430 */
    for (size_t j = 0; j < cols; ++j) y[j] = 0.0;
    for (size_t i = 0; i < rows; ++i) {
        double v = x[i];
        if (v == 0.0) continue;
        const double* ri = m + i * cols;
        for (size_t j = 0; j < cols; ++j) y[j] += v * ri[j];
    }
}

static uint64_t splitmix64(uint64_t x) { /* decomp.hpp:186-191 */
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

double orc_spectral_norm(const double* mat, size_t rows, size_t cols, double tol, size_t max_iter,
                         int* status, double* last_estimate) {
    /* decomp.hpp:206-239: power iteration on the smaller Gram operator */
    *status = ORC_OK;
    const double fro_sq = orc_frobenius_sq(mat, rows * cols);
    if (fro_sq == 0.0) {
        *status = ORC_DOMAIN_ERROR;
        return 0.0;
    }
    const int use_mtm = cols <= rows;
    const size_t dim = use_mtm ? cols : rows;
    const size_t other = use_mtm ? rows : cols;
    double* v = (double*)malloc(sizeof(double) * dim);
    double* w = (double*)malloc(sizeof(double) * dim);
    double* t = (double*)malloc(sizeof(double) * other);
    uint64_t h = 0x6b8f9a37c1d2e4f5ULL;
    for (size_t i = 0; i < dim; ++i) {
        h = splitmix64(h);
        v[i] = 1.0 + 1e-3 * ((double)(h >> 11) * 0x1.0p-53 - 0.5);
    }
    double nrm = 0.0; /* std::inner_product, sequential */
    for (size_t i = 0; i < dim; ++i) nrm = nrm + v[i] * v[i];
    nrm = sqrt(nrm);
    for (size_t i = 0; i < dim; ++i) v[i] /= nrm;

    double lambda = 0.0, result = 0.0;
    int done = 0;
    for (size_t it = 0; it < max_iter && !done; ++it) {
        /* gram_apply (decomp.hpp:193-200) */
        if (use_mtm) {
            matvec(mat, rows, cols, v, t);
            matvec_transposed(mat, rows, cols, t, w);
        } else {
            matvec_transposed(mat, rows, cols, v, t);
            matvec(mat, rows, cols, t, w);
        }
        double rayleigh = 0.0, wn = 0.0;
        for (size_t i = 0; i < dim; ++i) rayleigh = rayleigh + v[i] * w[i];
        for (size_t i = 0; i < dim; ++i) wn = wn + w[i] * w[i];
        wn = sqrt(wn);
        if (wn == 0.0) {
            result = 0.0;
            done = 1;
            break;
        }
        for (size_t i = 0; i < dim; ++i) v[i] = w[i] / wn;
        if (it > 0 && fabs(rayleigh - lambda) <= 0.5 * tol * fabs(rayleigh)) {
            result = sqrt(rayleigh);
            done = 1;
            break;
        }
        lambda = rayleigh;
    }
    free(v);
    free(w);
    free(t);
    if (!done) {
        *status = ORC_CONVERGENCE_ERROR;
        if (last_estimate) *last_estimate = sqrt(fabs(lambda));
        return 0.0;
    }
    return result;
}

void orc_generate_gaussian(uint64_t seed, size_t m, size_t p, size_t q, size_t n, double* A,
                           double* B, double* X, double* C) {
    /* problems.hpp:345-364 with GaussianSource for both A and B */
    orc_rng root, sa, sb, sx;
    orc_rng_init(&root, seed);
    orc_rng_substream(&root, 1, &sa);
    orc_rng_substream(&root, 2, &sb);
    orc_rng_substream(&root, 3, &sx);
    double* a = A ? A : (double*)malloc(sizeof(double) * m * p);
    double* b = B ? B : (double*)malloc(sizeof(double) * q * n);
    double* x = X ? X : (double*)malloc(sizeof(double) * p * q);
    orc_dense_gaussian(&sa, m, p, a);
    orc_dense_gaussian(&sb, q, n, b);
    orc_dense_gaussian(&sx, p, q, x);
    if (C) {
        double* t = (double*)malloc(sizeof(double) * m * q);
        orc_matmul(a, m, p, x, q, t);
        orc_matmul(t, m, q, b, n, C);
        free(t);
    }
    if (!A) free(a);
    if (!B) free(b);
    if (!X) free(x);
}

/* ------------------------------------------------------------------------ */
/* Solver<DenseMatrix,DenseMatrix> — solver.hpp:143-515                      */

struct orc_solver {
    size_t m, p, q, n;
    double *a, *b, *c, *x, *ref;
    orc_config cfg;
    orc_rng rng;
    double *gram, *btb, *r;
    double *a_sq, *r_sq, *rbk_cumsum;
    double a_fro_sq, r_fro_sq, r_fro_peak;
    double b_spec, alpha, c_fro;
    double ref_sq, err_sq;
    int alpha_outside_bound;
    size_t k, cyclic_pos, skipped_zero_rows;
    double *y, *z;
    size_t* members;
    double* member_cum;
    size_t n_members;
    int borrowed; /* A, B, C, gram, btb owned by the caller (prepared state) */
    /* error channel: C stand-in for the reference's exceptions */
    jmp_buf jb;
    int status;
    uint64_t div_k;
    double div_res;
    char err[256];
};

static void fail(orc_solver* s, int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(s->err, sizeof s->err, fmt, ap);
    va_end(ap);
    s->status = code;
    longjmp(s->jb, 1);
}

static double* dup(const double* src, size_t len) {
    double* d = (double*)malloc(sizeof(double) * (len ? len : 1));
    if (src) memcpy(d, src, sizeof(double) * len);
    else memset(d, 0, sizeof(double) * (len ? len : 1));
    return d;
}

static void row_sq_norms_of_r(orc_solver* s) { /* solver.hpp:458-466 */
    for (size_t i = 0; i < s->m; ++i) {
        const double* row = s->r + i * s->n;
        double acc = 0.0;
        for (size_t j = 0; j < s->n; ++j) acc += row[j] * row[j];
        s->r_sq[i] = acc;
    }
}

/* exact_residual (solver.hpp:420): C − (A·X)·B into out */
static void exact_residual(const orc_solver* s, double* out) {
    double* t = (double*)malloc(sizeof(double) * s->m * s->q);
    orc_matmul(s->a, s->m, s->p, s->x, s->q, t);
    orc_matmul(t, s->m, s->q, s->b, s->n, out);
    free(t);
    for (size_t i = 0; i < s->m * s->n; ++i) out[i] = s->c[i] - out[i]; /* sub(): matrix.hpp:594-601 */
}

static double frob_diff_sq(const double* a, const double* b, size_t len) {
    /* frobenius_sq(sub(a, b)) — matrix.hpp:594-601 then :276-280 */
    double acc = 0.0;
    for (size_t i = 0; i < len; ++i) {
        double d = a[i] - b[i];
        acc += d * d;
    }
    return acc;
}

static void adopt_residual(orc_solver* s, double* exact) { /* solver.hpp:468-476 */
    free(s->r);
    s->r = exact;
    row_sq_norms_of_r(s);
    s->r_fro_sq = 0.0;
    for (size_t i = 0; i < s->m; ++i) s->r_fro_sq += s->r_sq[i];
    s->r_fro_peak = s->r_fro_sq;
    if (s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN)
        s->err_sq = frob_diff_sq(s->x, s->ref, s->p * s->q);
}

static void resolve_alpha(orc_solver* s) { /* solver.hpp:439-456 */
    const double b2 = s->b_spec * s->b_spec;
    switch (s->cfg.alpha_rule) {
        case ORC_ALPHA_SAFE: s->alpha = 1.0 / b2; break;
        case ORC_ALPHA_PAPER:
            s->alpha = 1.0 / s->b_spec;
            s->alpha_outside_bound = !(s->alpha < 2.0 / b2);
            break;
        case ORC_ALPHA_FIXED:
            s->alpha = s->cfg.alpha_value;
            if (!(s->alpha > 0.0) || !(s->alpha < 2.0 / b2))
                fail(s, ORC_CONFIG_ERROR, "fixed alpha %f outside (0, 2/|B|_2^2)", s->alpha);
            break;
        default: fail(s, ORC_CONFIG_ERROR, "unknown alpha rule");
    }
}

static void validate_method(orc_solver* s) { /* solver.hpp:30-38 */
    if (s->cfg.method < ORC_BK || s->cfg.method > ORC_MWRBK)
        fail(s, ORC_CONFIG_ERROR, "unknown method");
    if (s->cfg.method == ORC_RGRBK) {
        if (!s->cfg.has_theta) fail(s, ORC_CONFIG_ERROR, "rgrbk requires theta");
        if (!(s->cfg.theta > 0.0 && s->cfg.theta < 1.0))
            fail(s, ORC_CONFIG_ERROR, "theta must lie strictly in (0, 1)");
    } else if (s->cfg.has_theta) {
        fail(s, ORC_CONFIG_ERROR, "theta is only valid for rgrbk");
    }
}

static void solver_init(orc_solver* s) { /* solver.hpp:146-192 */
    validate_method(s);
    const size_t m = s->m, p = s->p, q = s->q, n = s->n;
    if (m == 0 || p == 0) fail(s, ORC_SHAPE_ERROR, "row_sq_norms: empty matrix");
    /* a_sq_ = row_sq_norms(A) : matrix.hpp:300-306 via RowView::sq_norm :199-203 */
    for (size_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (size_t j = 0; j < p; ++j) acc += s->a[i * p + j] * s->a[i * p + j];
        s->a_sq[i] = acc;
    }
    s->a_fro_sq = 0.0;
    for (size_t i = 0; i < m; ++i) s->a_fro_sq += s->a_sq[i];
    if (s->a_fro_sq == 0.0) fail(s, ORC_DOMAIN_ERROR, "solve: A is the zero matrix");
    double cum = 0.0;
    for (size_t i = 0; i < m; ++i) {
        cum += s->a_sq[i];
        s->rbk_cumsum[i] = cum;
    }
    int st = 0;
    double last = 0.0;
    s->b_spec = orc_spectral_norm(s->b, q, n, 1e-10, 5000, &st, &last);
    if (st == ORC_DOMAIN_ERROR) fail(s, st, "spectral_norm: zero matrix");
    if (st == ORC_CONVERGENCE_ERROR)
        fail(s, st, "spectral_norm: power iteration did not converge (last %.17g)", last);
    resolve_alpha(s);

    orc_gram_mmt(s->a, m, p, s->gram);
    /* btb_ = matmul(transpose(B), B) */
    double* bt = (double*)malloc(sizeof(double) * q * n);
    for (size_t i = 0; i < q; ++i)
        for (size_t j = 0; j < n; ++j) bt[j * q + i] = s->b[i * n + j];
    orc_matmul(bt, n, q, s->b, n, s->btb);
    free(bt);
    exact_residual(s, s->r);
    row_sq_norms_of_r(s);
    s->r_fro_sq = 0.0;
    for (size_t i = 0; i < m; ++i) s->r_fro_sq += s->r_sq[i];
    s->r_fro_peak = s->r_fro_sq;
    s->c_fro = sqrt(orc_frobenius_sq(s->c, m * n));
    if (s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN) {
        if (!s->ref) fail(s, ORC_CONFIG_ERROR, "solution_rrn stopping needs a reference solution");
        s->ref_sq = orc_frobenius_sq(s->ref, p * q);
        if (s->ref_sq == 0.0) fail(s, ORC_DOMAIN_ERROR, "solution_rrn: zero reference");
        s->err_sq = frob_diff_sq(s->x, s->ref, p * q);
    }
}

orc_solver* orc_solver_create(const double* A, size_t m, size_t p, const double* B, size_t q,
                              size_t n, const double* C, const double* X0, const orc_config* cfg,
                              int* status, char* errbuf, size_t errlen) {
    orc_solver* s = (orc_solver*)calloc(1, sizeof(orc_solver));
    s->m = m; s->p = p; s->q = q; s->n = n;
    s->cfg = *cfg;
    s->a = dup(A, m * p);
    s->b = dup(B, q * n);
    s->c = dup(C, m * n);
    s->x = dup(X0, p * q);
    s->ref = cfg->reference ? dup(cfg->reference, p * q) : NULL;
    s->cfg.reference = s->ref;
    orc_rng_init(&s->rng, cfg->seed);
    s->gram = dup(NULL, m * m);
    s->btb = dup(NULL, n * n);
    s->r = dup(NULL, m * n);
    s->a_sq = dup(NULL, m);
    s->r_sq = dup(NULL, m);
    s->rbk_cumsum = dup(NULL, m);
    s->y = dup(NULL, q);
    s->z = dup(NULL, n);
    s->members = (size_t*)malloc(sizeof(size_t) * (m ? m : 1));
    s->member_cum = dup(NULL, m);
    if (setjmp(s->jb)) {
        if (status) *status = s->status;
        if (errbuf && errlen) snprintf(errbuf, errlen, "%s", s->err);
        orc_solver_destroy(s);
        return NULL;
    }
    solver_init(s);
    if (status) *status = ORC_OK;
    return s;
}

void orc_solver_destroy(orc_solver* s) {
    if (!s) return;
    if (!s->borrowed) {
        free(s->a); free(s->b); free(s->c);
        free(s->gram); free(s->btb);
    }
    free(s->x); free(s->ref); free(s->r);
    free(s->a_sq); free(s->r_sq); free(s->rbk_cumsum);
    free(s->y); free(s->z); free(s->members); free(s->member_cum);
    free(s);
}

const char* orc_solver_last_error(const orc_solver* s) { return s->err; }

/* -- selection rules (solver.hpp:197-258, 387-400) -- */

static size_t select_cyclic(orc_solver* s) { /* :197-206 */
    for (size_t tries = 0; tries < s->m; ++tries) {
        size_t i = s->cyclic_pos;
        s->cyclic_pos = (s->cyclic_pos + 1) % s->m;
        if (s->a_sq[i] > 0.0) return i;
        ++s->skipped_zero_rows;
    }
    fail(s, ORC_DOMAIN_ERROR, "select_cyclic: no nonzero row");
    return 0;
}

static size_t select_rbk(orc_solver* s) { /* :209 */
    int st = 0;
    size_t i = orc_rng_categorical_cdf(&s->rng, s->rbk_cumsum, s->m, &st);
    if (st) fail(s, st, "categorical: no positive weight");
    return i;
}

static void max_residual_ratio(orc_solver* s, size_t* best_out, double* ratio_out) { /* :387-400 */
    size_t best = s->m;
    double best_ratio = -INFINITY;
    for (size_t i = 0; i < s->m; ++i) {
        if (s->a_sq[i] <= 0.0) continue;
        const double ratio = s->r_sq[i] / s->a_sq[i];
        if (ratio > best_ratio) {
            best_ratio = ratio;
            best = i;
        }
    }
    if (best == s->m) fail(s, ORC_DOMAIN_ERROR, "no nonzero row in A");
    *best_out = best;
    *ratio_out = best_ratio;
}

static double greedy_threshold(orc_solver* s, double theta) { /* :212-216 */
    if (!(s->r_fro_sq > 0.0)) fail(s, ORC_DOMAIN_ERROR, "greedy threshold: zero residual");
    size_t best;
    double max_ratio;
    max_residual_ratio(s, &best, &max_ratio);
    return theta * (max_ratio / s->r_fro_sq) + (1.0 - theta) / s->a_fro_sq;
}

static void greedy_index_set(orc_solver* s, double theta) { /* :226-237 */
    const double zeta = greedy_threshold(s, theta);
    size_t argmax_row;
    double ratio;
    max_residual_ratio(s, &argmax_row, &ratio);
    s->n_members = 0;
    for (size_t i = 0; i < s->m; ++i) {
        if (s->a_sq[i] <= 0.0) continue;
        if (i == argmax_row || s->r_sq[i] >= zeta * s->a_sq[i] * s->r_fro_sq)
            s->members[s->n_members++] = i;
    }
    if (s->n_members == 0) fail(s, ORC_INVARIANT_ERROR, "greedy index set is empty");
}

static size_t select_greedy(orc_solver* s, double theta) { /* :241-254 */
    greedy_index_set(s, theta);
    double cum = 0.0;
    for (size_t k = 0; k < s->n_members; ++k) {
        cum += s->r_sq[s->members[k]];
        s->member_cum[k] = cum;
    }
    if (!(cum > 0.0))
        fail(s, ORC_DOMAIN_ERROR,
             "greedy selection: residual mass sits on zero rows of A only; the system is "
             "inconsistent");
    int st = 0;
    size_t idx = orc_rng_categorical_cdf(&s->rng, s->member_cum, s->n_members, &st);
    if (st) fail(s, st, "categorical: no positive weight");
    return s->members[idx];
}

static size_t select_mwrbk(orc_solver* s) { /* :258 */
    size_t best;
    double ratio;
    max_residual_ratio(s, &best, &ratio);
    return best;
}

/* -- kernel: update_row (solver.hpp:264-318) -- */
static void update_row(orc_solver* s, size_t i) {
    if (!(s->a_sq[i] > 0.0)) fail(s, ORC_DOMAIN_ERROR, "update_row: zero row selected");
    const size_t p = s->p, q = s->q, n = s->n, m = s->m;
    const double coef = s->alpha / s->a_sq[i];
    const double* r_i = s->r + i * n;
    matvec(s->b, q, n, r_i, s->y); /* y = R_i Bᵀ (:270) */
    const int track = s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN;
    for (size_t t = 0; t < p; ++t) { /* RowView(A,i).for_each over dense row: every column */
        const double v = s->a[i * p + t];
        const double f = coef * v;
        double* xrow = s->x + t * q;
        if (track) {
            const double* ref_row = s->ref + t * q;
            double delta = 0.0;
            for (size_t j = 0; j < q; ++j) {
                const double d0 = xrow[j] - ref_row[j];
                xrow[j] += f * s->y[j];
                const double d1 = xrow[j] - ref_row[j];
                delta += d1 * d1 - d0 * d0;
            }
            s->err_sq += delta;
        } else {
            for (size_t j = 0; j < q; ++j) xrow[j] += f * s->y[j];
        }
    }
    if (s->err_sq < 0.0) s->err_sq = 0.0;

    matvec(s->btb, n, n, r_i, s->z); /* z = R_i BᵀB (:293) */
    for (size_t l = 0; l < m; ++l) { /* dense G row: every column (:294-305) */
        const double g = s->gram[i * m + l];
        const double f = coef * g;
        double* rrow = s->r + l * n;
        double ns = 0.0;
        for (size_t j = 0; j < n; ++j) {
            rrow[j] -= f * s->z[j];
            ns += rrow[j] * rrow[j];
        }
        s->r_fro_sq += ns - s->r_sq[l];
        s->r_sq[l] = ns;
    }
    if (s->r_fro_sq < 0.0) s->r_fro_sq = 0.0;
    if (!isfinite(s->r_fro_sq)) {
        s->div_k = s->k;
        s->div_res = sqrt(fabs(s->r_fro_sq));
        fail(s, ORC_DIVERGENCE_ERROR, "divergence at iteration %llu, residual frobenius norm %f",
             (unsigned long long)s->k, s->div_res);
    }
    if (s->r_fro_sq < 1e-12 * s->r_fro_peak) { /* :311-317 */
        s->r_fro_sq = 0.0;
        for (size_t l = 0; l < m; ++l) s->r_fro_sq += s->r_sq[l];
        s->r_fro_peak = s->r_fro_sq;
    } else if (s->r_fro_sq > s->r_fro_peak) {
        s->r_fro_peak = s->r_fro_sq;
    }
}

static size_t step(orc_solver* s) { /* :321-333 */
    size_t i = 0;
    switch (s->cfg.method) {
        case ORC_BK: i = select_cyclic(s); break;
        case ORC_RBK: i = select_rbk(s); break;
        case ORC_GRBK: i = select_greedy(s, 0.5); break;
        case ORC_RGRBK: i = select_greedy(s, s->cfg.theta); break;
        case ORC_MWRBK: i = select_mwrbk(s); break;
    }
    update_row(s, i);
    ++s->k;
    return i;
}

double orc_solver_current_residual_rel(const orc_solver* s) { /* :407-409 */
    return sqrt(s->r_fro_sq > 0.0 ? s->r_fro_sq : 0.0) / (s->c_fro > 0.0 ? s->c_fro : 1.0);
}

double orc_solver_current_metric(const orc_solver* s) { /* :403-406 */
    if (s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN) return s->err_sq / s->ref_sq;
    return orc_solver_current_residual_rel(s);
}

static double exact_residual_rel(orc_solver* s) { /* :417-419 */
    double* e = (double*)malloc(sizeof(double) * s->m * s->n);
    exact_residual(s, e);
    double v = sqrt(orc_frobenius_sq(e, s->m * s->n)) / (s->c_fro > 0.0 ? s->c_fro : 1.0);
    free(e);
    return v;
}

static double exact_metric(orc_solver* s) { /* :412-416 */
    if (s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN)
        return frob_diff_sq(s->x, s->ref, s->p * s->q) / s->ref_sq;
    return exact_residual_rel(s);
}

static void resync(orc_solver* s) { /* :478 */
    double* e = (double*)malloc(sizeof(double) * s->m * s->n);
    exact_residual(s, e);
    adopt_residual(s, e);
}

static int all_finite(const double* a, size_t len) {
    for (size_t i = 0; i < len; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

static void checkpoint(orc_solver* s) { /* :427-436 */
    if (!all_finite(s->x, s->p * s->q)) {
        s->div_k = s->k;
        s->div_res = sqrt(s->r_fro_sq > 0.0 ? s->r_fro_sq : 0.0);
        fail(s, ORC_DIVERGENCE_ERROR, "divergence at iteration %llu", (unsigned long long)s->k);
    }
    double* e = (double*)malloc(sizeof(double) * s->m * s->n);
    exact_residual(s, e);
    const double drift = sqrt(frob_diff_sq(s->r, e, s->m * s->n));
    if (drift > 1e-8 * (1.0 + s->c_fro)) {
        free(e);
        fail(s, ORC_INVARIANT_ERROR, "residual drift guard tripped at iteration %llu",
             (unsigned long long)s->k);
    }
    adopt_residual(s, e);
}

/* ---- public wrappers: setjmp around each throwing entry point ---- */
#define GUARD(s)                 \
    do {                         \
        (s)->status = ORC_OK;    \
        if (setjmp((s)->jb)) return (s)->status; \
    } while (0)

int orc_solver_step(orc_solver* s, uint64_t* row) { GUARD(s); *row = step(s); return 0; }
int orc_solver_update_row(orc_solver* s, uint64_t i) {
    GUARD(s);
    if (i >= s->m) fail(s, ORC_SHAPE_ERROR, "row out of range");
    update_row(s, i);
    return 0;
}
int orc_solver_select_cyclic(orc_solver* s, uint64_t* row) { GUARD(s); *row = select_cyclic(s); return 0; }
int orc_solver_select_rbk(orc_solver* s, uint64_t* row) { GUARD(s); *row = select_rbk(s); return 0; }
int orc_solver_select_greedy(orc_solver* s, double theta, uint64_t* row) {
    GUARD(s); *row = select_greedy(s, theta); return 0;
}
int orc_solver_select_mwrbk(orc_solver* s, uint64_t* row) { GUARD(s); *row = select_mwrbk(s); return 0; }
int orc_solver_greedy_threshold(orc_solver* s, double theta, double* out) {
    GUARD(s); *out = greedy_threshold(s, theta); return 0;
}
int orc_solver_rgrbk_threshold(orc_solver* s, double theta, double* out) { /* :218-221 */
    GUARD(s);
    if (!(theta > 0.0 && theta < 1.0)) fail(s, ORC_CONFIG_ERROR, "theta must lie in (0, 1)");
    *out = greedy_threshold(s, theta);
    return 0;
}
int orc_solver_greedy_index_set(orc_solver* s, double theta, uint64_t* out, uint64_t* count) {
    GUARD(s);
    greedy_index_set(s, theta);
    for (size_t k = 0; k < s->n_members; ++k) out[k] = s->members[k];
    *count = s->n_members;
    return 0;
}
int orc_solver_max_residual_ratio(orc_solver* s, uint64_t* row, double* ratio) {
    GUARD(s);
    size_t b;
    max_residual_ratio(s, &b, ratio);
    *row = b;
    return 0;
}
int orc_solver_checkpoint(orc_solver* s) { GUARD(s); checkpoint(s); return 0; }
int orc_solver_exact_metric(orc_solver* s, double* out) { GUARD(s); *out = exact_metric(s); return 0; }
int orc_solver_exact_residual_rel(orc_solver* s, double* out) {
    GUARD(s); *out = exact_residual_rel(s); return 0;
}
int orc_solver_residual_drift(orc_solver* s, double* out) { /* :423 */
    GUARD(s);
    double* e = (double*)malloc(sizeof(double) * s->m * s->n);
    exact_residual(s, e);
    *out = sqrt(frob_diff_sq(s->r, e, s->m * s->n));
    free(e);
    return 0;
}

static int trace_point_due(size_t k) { return k < 10000 || k % 10 == 0; } /* solver.hpp:136 */

int orc_solver_run(orc_solver* s, orc_report* rep, uint64_t* trace_k, double* trace_rrn,
                   double* trace_rel, uint64_t* trace_row, uint64_t trace_cap, double* x_out) {
    /* solver.hpp:337-372 */
    memset(rep, 0, sizeof *rep);
    rep->alpha = s->alpha;
    rep->seed = s->cfg.seed;
    rep->alpha_outside_bound = s->alpha_outside_bound;
    s->status = ORC_OK;
    if (setjmp(s->jb)) {
        rep->iterations = s->k;
        rep->diverged_iteration = s->div_k;
        rep->diverged_residual = s->div_res;
        return s->status;
    }
    int converged = exact_metric(s) <= s->cfg.tol;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    uint64_t ntrace = 0;
    while (!converged && s->k < s->cfg.max_iter) {
        if (!(s->r_fro_sq > 0.0)) break;
        const size_t i = step(s);
        if (s->cfg.record_trace && trace_point_due(s->k - 1)) {
            if (ntrace < trace_cap) {
                if (trace_k) trace_k[ntrace] = s->k - 1;
                if (trace_rrn) trace_rrn[ntrace] = orc_solver_current_metric(s);
                if (trace_rel) trace_rel[ntrace] = orc_solver_current_residual_rel(s);
                if (trace_row) trace_row[ntrace] = i;
            }
            ++ntrace;
        }
        if (orc_solver_current_metric(s) <= s->cfg.tol) {
            if (exact_metric(s) <= s->cfg.tol)
                converged = 1;
            else
                resync(s);
        }
        if (!converged && s->cfg.refresh_interval > 0 && s->k % s->cfg.refresh_interval == 0)
            checkpoint(s);
    }
    clock_gettime(CLOCK_MONOTONIC, &t1);
    rep->iterations = s->k;
    rep->wall_seconds = (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    rep->terminated_by = converged ? 0 : 1;
    rep->final_rrn = exact_metric(s);
    rep->final_residual_rel = exact_residual_rel(s);
    rep->skipped_zero_rows = s->skipped_zero_rows;
    rep->trace_len = ntrace;
    if (x_out) memcpy(x_out, s->x, sizeof(double) * s->p * s->q);
    return 0;
}

uint64_t orc_solver_iteration(const orc_solver* s) { return s->k; }
double orc_solver_alpha(const orc_solver* s) { return s->alpha; }
double orc_solver_spectral_norm_b(const orc_solver* s) { return s->b_spec; }
int orc_solver_alpha_outside_bound(const orc_solver* s) { return s->alpha_outside_bound; }
double orc_solver_a_fro_sq(const orc_solver* s) { return s->a_fro_sq; }
double orc_solver_residual_fro_sq(const orc_solver* s) { return s->r_fro_sq; }
void orc_solver_get_X(const orc_solver* s, double* out) { memcpy(out, s->x, sizeof(double) * s->p * s->q); }
void orc_solver_get_R(const orc_solver* s, double* out) { memcpy(out, s->r, sizeof(double) * s->m * s->n); }
void orc_solver_get_r_sq(const orc_solver* s, double* out) { memcpy(out, s->r_sq, sizeof(double) * s->m); }
void orc_solver_get_a_sq(const orc_solver* s, double* out) { memcpy(out, s->a_sq, sizeof(double) * s->m); }
void orc_solver_rng_state(const orc_solver* s, uint64_t out[4]) { memcpy(out, s->rng.s, 32); }

/* ------------------------------------------------------------------------ */
/* Prepared state (benchmark only): the caches the reference constructor builds
 * sequentially (gram_mmt, BᵀB, C − A·X0·B: ~10¹² flops at config-3 size, ~400 s
 * on one core) are supplied by the caller and BORROWED; everything else follows
 * solver.hpp:146-192.  The per-iteration algorithm timed afterwards is exactly
 * step() → select_* + update_row (solver.hpp:197-333). */
orc_solver* orc_solver_create_prepared(const double* A, size_t m, size_t p, const double* B,
                                       size_t q, size_t n, const double* C, const double* X0,
                                       const double* R0, const double* G, const double* BtB,
                                       double alpha, const orc_config* cfg, int* status) {
    orc_solver* s = (orc_solver*)calloc(1, sizeof(orc_solver));
    s->m = m; s->p = p; s->q = q; s->n = n;
    s->cfg = *cfg;
    s->borrowed = 1;
    s->a = (double*)A; s->b = (double*)B; s->c = (double*)C;
    s->gram = (double*)G; s->btb = (double*)BtB;
    s->x = dup(X0, p * q);
    s->ref = cfg->reference ? dup(cfg->reference, p * q) : NULL;
    s->cfg.reference = s->ref;
    s->r = dup(R0, m * n);
    orc_rng_init(&s->rng, cfg->seed);
    s->a_sq = dup(NULL, m); s->r_sq = dup(NULL, m); s->rbk_cumsum = dup(NULL, m);
    s->y = dup(NULL, q); s->z = dup(NULL, n);
    s->members = (size_t*)malloc(sizeof(size_t) * (m ? m : 1));
    s->member_cum = dup(NULL, m);
    if (setjmp(s->jb)) {
        if (status) *status = s->status;
        orc_solver_destroy(s);
        return NULL;
    }
    validate_method(s);
    for (size_t i = 0; i < m; ++i) {
        double acc = 0.0;
        for (size_t j = 0; j < p; ++j) acc += s->a[i * p + j] * s->a[i * p + j];
        s->a_sq[i] = acc;
    }
    s->a_fro_sq = 0.0;
    for (size_t i = 0; i < m; ++i) s->a_fro_sq += s->a_sq[i];
    double cum = 0.0;
    for (size_t i = 0; i < m; ++i) { cum += s->a_sq[i]; s->rbk_cumsum[i] = cum; }
    s->alpha = alpha;
    row_sq_norms_of_r(s);
    s->r_fro_sq = 0.0;
    for (size_t i = 0; i < m; ++i) s->r_fro_sq += s->r_sq[i];
    s->r_fro_peak = s->r_fro_sq;
    s->c_fro = sqrt(orc_frobenius_sq(s->c, m * n));
    if (s->cfg.stop_kind == ORC_STOP_SOLUTION_RRN && s->ref) {
        s->ref_sq = orc_frobenius_sq(s->ref, p * q);
        s->err_sq = frob_diff_sq(s->x, s->ref, p * q);
    }
    if (status) *status = ORC_OK;
    return s;
}

/* k consecutive step() calls in C (no interpreter in the loop; ctypes releases
 * the GIL, so several solvers can run on several cores concurrently — the
 * reference benchmark pool pattern, analysis.hpp:295-313). */
int orc_solver_steps(orc_solver* s, uint64_t k, uint64_t* rows) {
    GUARD(s);
    for (uint64_t t = 0; t < k; ++t) {
        size_t i = step(s);
        if (rows) rows[t] = i;
    }
    return 0;
}

/* ======================================================================== */
/* Reference solutions: decomp.hpp + analysis.hpp             */
/* ======================================================================== */

static int set_err(char* err, int code, const char* msg) {
    if (err) snprintf(err, 256, "%s", msg);
    return code;
}

static double* transposed(const double* a, size_t rows, size_t cols) { /* matrix.hpp:448-453 */
    double* t = (double*)malloc(sizeof(double) * (rows * cols ? rows * cols : 1));
    for (size_t i = 0; i < rows; ++i)
        for (size_t j = 0; j < cols; ++j) t[j * rows + i] = a[i * cols + j];
    return t;
}

static double* mm(const double* a, size_t ar, size_t ac, const double* b, size_t bc) {
    double* c = (double*)malloc(sizeof(double) * (ar * bc ? ar * bc : 1));
    orc_matmul(a, ar, ac, b, bc, c);
    return c;
}

static double default_rank_tol(size_t rows, size_t cols, double sigma_max) { /* decomp.hpp:30-33 */
    return 8.0 * (double)(rows > cols ? rows : cols) * sigma_max * ldexp(1.0, -52);
}

/* detail::complete_orthonormal_columns (decomp.hpp:39-65); u is m×r */
static int complete_orthonormal_columns(double* u, size_t m, size_t r, size_t from) {
    size_t next_basis = 0;
    double* cand = (double*)malloc(sizeof(double) * (m ? m : 1));
    for (size_t j = from; j < r; ++j) {
        for (; next_basis <= m; ++next_basis) {
            if (next_basis == m) {
                free(cand);
                return -1;
            }
            memset(cand, 0, sizeof(double) * m);
            cand[next_basis] = 1.0;
            for (int pass = 0; pass < 2; ++pass) { /* twice-is-enough Gram-Schmidt */
                for (size_t c = 0; c < j; ++c) {
                    double dot = 0.0;
                    for (size_t i = 0; i < m; ++i) dot += cand[i] * u[i * r + c];
                    for (size_t i = 0; i < m; ++i) cand[i] -= dot * u[i * r + c];
                }
            }
            double nrm = 0.0;
            for (size_t i = 0; i < m; ++i) nrm += cand[i] * cand[i];
            nrm = sqrt(nrm);
            if (nrm > 0.5) {
                for (size_t i = 0; i < m; ++i) u[i * r + j] = cand[i] / nrm;
                ++next_basis;
                break;
            }
        }
    }
    free(cand);
    return 0;
}

/* detail::jacobi_factor (decomp.hpp:71-109): one-sided cyclic Jacobi on w (m×n,
 * m >= n), right rotations accumulated into v (n×n); -1 when the cap is hit */
static int jacobi_factor(double* w, size_t m, size_t n, double* v, size_t max_sweeps) {
    const double tol = 1e-15;
    const double null_sq = orc_frobenius_sq(w, m * n) * 1e-30;
    for (size_t sweep = 0; sweep < max_sweeps; ++sweep) {
        int rotated = 0;
        for (size_t p = 0; p + 1 < n; ++p) {
            for (size_t q = p + 1; q < n; ++q) {
                double app = 0.0, aqq = 0.0, apq = 0.0;
                for (size_t i = 0; i < m; ++i) {
                    double wp = w[i * n + p], wq = w[i * n + q];
                    app += wp * wp;
                    aqq += wq * wq;
                    apq += wp * wq;
                }
                if (app <= null_sq || aqq <= null_sq) continue;
                if (fabs(apq) <= tol * sqrt(app * aqq)) continue;
                rotated = 1;
                double zeta = (aqq - app) / (2.0 * apq);
                double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                double c = 1.0 / sqrt(1.0 + t * t);
                double s = c * t;
                for (size_t i = 0; i < m; ++i) {
                    double wp = w[i * n + p], wq = w[i * n + q];
                    w[i * n + p] = c * wp - s * wq;
                    w[i * n + q] = s * wp + c * wq;
                }
                for (size_t i = 0; i < n; ++i) {
                    double vp = v[i * n + p], vq = v[i * n + q];
                    v[i * n + p] = c * vp - s * vq;
                    v[i * n + q] = s * vp + c * vq;
                }
            }
        }
        if (!rotated) return 0;
    }
    return -1;
}

int orc_svd(const double* M, size_t rows, size_t cols, size_t max_sweeps, double* U_out,
            double* sigma_out, double* V_out, size_t* rank_out, char* err) {
    if (rows == 0 || cols == 0) return set_err(err, ORC_SHAPE_ERROR, "svd: empty matrix");
    const int wide = rows < cols;
    double* w = wide ? transposed(M, rows, cols) : dup(M, rows * cols);
    const size_t m = wide ? cols : rows, n = wide ? rows : cols;
    double* v = (double*)calloc(n * n, sizeof(double));
    for (size_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
    if (jacobi_factor(w, m, n, v, max_sweeps) != 0) {
        free(w);
        free(v);
        return set_err(err, ORC_DECOMPOSITION_ERROR, "svd: Jacobi sweeps exceeded cap");
    }
    double* sigma = (double*)malloc(sizeof(double) * n);
    for (size_t j = 0; j < n; ++j) {
        double s = 0.0;
        for (size_t i = 0; i < m; ++i) s += w[i * n + j] * w[i * n + j];
        sigma[j] = sqrt(s);
    }
    size_t* order = (size_t*)malloc(sizeof(size_t) * n);
    for (size_t j = 0; j < n; ++j) { /* std::stable_sort by sigma, descending */
        size_t k = j;
        while (k > 0 && sigma[order[k - 1]] < sigma[j]) {
            order[k] = order[k - 1];
            --k;
        }
        order[k] = j;
    }
    double* sv = (double*)malloc(sizeof(double) * n);
    double* fU = (double*)calloc(m * n, sizeof(double));
    double* fV = (double*)malloc(sizeof(double) * n * n);
    for (size_t j = 0; j < n; ++j) {
        size_t src = order[j];
        sv[j] = sigma[src];
        for (size_t i = 0; i < n; ++i) fV[i * n + j] = v[i * n + src];
    }
    const double cutoff = default_rank_tol(rows, cols, sv[0]);
    size_t solid = 0;
    for (size_t j = 0; j < n; ++j) {
        size_t src = order[j];
        if (sv[j] > cutoff) {
            for (size_t i = 0; i < m; ++i) fU[i * n + j] = w[i * n + src] / sv[j];
            solid = j + 1;
        }
    }
    int rc = complete_orthonormal_columns(fU, m, n, solid);
    if (rc == 0) {
        /* tall: U = fU (rows×n), V = fV (cols×n); wide: swapped */
        const double* u = wide ? fV : fU;
        const double* vv = wide ? fU : fV;
        if (U_out) memcpy(U_out, u, sizeof(double) * rows * n);
        if (V_out) memcpy(V_out, vv, sizeof(double) * cols * n);
        if (sigma_out) memcpy(sigma_out, sv, sizeof(double) * n);
        if (rank_out) *rank_out = solid;
    }
    free(w); free(v); free(sigma); free(order); free(sv); free(fU); free(fV);
    if (rc != 0) return set_err(err, ORC_DECOMPOSITION_ERROR, "svd: failed to complete orthonormal basis");
    return ORC_OK;
}

int orc_pseudoinverse(const double* M, size_t rows, size_t cols, double rank_tol, double* P,
                      char* err) {
    if (rows == 0 || cols == 0) return set_err(err, ORC_SHAPE_ERROR, "svd: empty matrix");
    const size_t r = rows < cols ? rows : cols;
    double* U = (double*)malloc(sizeof(double) * rows * r);
    double* V = (double*)malloc(sizeof(double) * cols * r);
    double* sv = (double*)malloc(sizeof(double) * r);
    int rc = orc_svd(M, rows, cols, 64, U, sv, V, NULL, err);
    if (rc == ORC_OK) {
        if (rank_tol < 0.0) rank_tol = default_rank_tol(rows, cols, sv[0]);
        memset(P, 0, sizeof(double) * cols * rows);
        for (size_t k = 0; k < r; ++k) {
            double s = sv[k];
            if (s <= rank_tol) continue;
            double inv = 1.0 / s;
            for (size_t i = 0; i < cols; ++i) {
                double vik = V[i * r + k] * inv;
                if (vik == 0.0) continue;
                for (size_t j = 0; j < rows; ++j) P[i * rows + j] += vik * U[j * r + k];
            }
        }
    }
    free(U); free(V); free(sv);
    return rc;
}

int orc_lu_solve(double* a, size_t n, double* b, size_t k, char* err) {
    for (size_t col = 0; col < n; ++col) {
        size_t piv = col;
        for (size_t i = col + 1; i < n; ++i)
            if (fabs(a[i * n + col]) > fabs(a[piv * n + col])) piv = i;
        if (a[piv * n + col] == 0.0)
            return set_err(err, ORC_DECOMPOSITION_ERROR, "lu_solve: singular matrix");
        if (piv != col) {
            for (size_t j = 0; j < n; ++j) {
                double t = a[col * n + j]; a[col * n + j] = a[piv * n + j]; a[piv * n + j] = t;
            }
            for (size_t j = 0; j < k; ++j) {
                double t = b[col * k + j]; b[col * k + j] = b[piv * k + j]; b[piv * k + j] = t;
            }
        }
        double d = a[col * n + col];
        for (size_t i = col + 1; i < n; ++i) {
            double f = a[i * n + col] / d;
            if (f == 0.0) continue;
            for (size_t j = col; j < n; ++j) a[i * n + j] -= f * a[col * n + j];
            for (size_t j = 0; j < k; ++j) b[i * k + j] -= f * b[col * k + j];
        }
    }
    for (size_t col = n; col-- > 0;) {
        double d = a[col * n + col];
        for (size_t j = 0; j < k; ++j) {
            double s = b[col * k + j];
            for (size_t t = col + 1; t < n; ++t) s -= a[col * n + t] * b[t * k + j];
            b[col * k + j] = s / d;
        }
    }
    return ORC_OK;
}

/* detail::right_solve_sym (analysis.hpp:39-41): x·m⁻¹ = (m⁻¹ᵀ... via lu_solve(m, xᵀ))ᵀ;
 * x is r×c, m c×c (consumed); result r×c in a new buffer */
static double* right_solve_sym(const double* x, size_t r, size_t c, double* msq, int* rc,
                               char* err) {
    double* xt = transposed(x, r, c);
    *rc = orc_lu_solve(msq, c, xt, r, err);
    double* out = transposed(xt, c, r);
    free(xt);
    return out;
}

int orc_reference_solution(const double* A, size_t m, size_t p, const double* B, size_t q,
                           size_t n, const double* C, double rank_tol, double* X, int* kind,
                           double* residual_check, char* err) {
    if (!m || !p || !q || !n) return set_err(err, ORC_SHAPE_ERROR, "svd: empty matrix");
    const size_t ra = m < p ? m : p, rb = q < n ? q : n;
    double* sa = (double*)malloc(sizeof(double) * ra);
    double* sb = (double*)malloc(sizeof(double) * rb);
    size_t rank_a = 0, rank_b = 0;
    int rc = orc_svd(A, m, p, 64, NULL, sa, NULL, &rank_a, err);
    if (rc == ORC_OK) rc = orc_svd(B, q, n, 64, NULL, sb, NULL, &rank_b, err);
    if (rc != ORC_OK) {
        free(sa); free(sb);
        return rc;
    }
    if (rank_tol >= 0.0) { /* rank_of (analysis.hpp:54-61) */
        rank_a = rank_b = 0;
        for (size_t k = 0; k < ra; ++k) rank_a += sa[k] > rank_tol;
        for (size_t k = 0; k < rb; ++k) rank_b += sb[k] > rank_tol;
    }
    free(sa); free(sb);
    const int a_full_col = rank_a == p, a_full_row = rank_a == m;
    const int b_full_col = rank_b == n, b_full_row = rank_b == q;
    double* At = transposed(A, m, p);
    double* Bt = transposed(B, q, n);
    double* xs = NULL;
    if (a_full_col && b_full_row) {
        /* (AᵀA)⁻¹ Aᵀ C Bᵀ (BBᵀ)⁻¹ (analysis.hpp:70-75) */
        double* ata = mm(At, p, m, A, p);
        double* atc = mm(At, p, m, C, n);
        double* y = mm(atc, p, n, Bt, q);
        free(atc);
        rc = orc_lu_solve(ata, p, y, q, err);
        free(ata);
        if (rc == ORC_OK) {
            double* bbt = mm(B, q, n, Bt, q);
            xs = right_solve_sym(y, p, q, bbt, &rc, err);
            free(bbt);
        }
        free(y);
        if (kind) *kind = ORC_REF_UNIQUE_FULL_RANK;
    } else if (a_full_row && b_full_col) {
        /* Aᵀ (AAᵀ)⁻¹ C (BᵀB)⁻¹ Bᵀ (analysis.hpp:76-81) */
        double* aat = mm(A, m, p, At, m);
        double* w = dup(C, m * n);
        rc = orc_lu_solve(aat, m, w, n, err);
        free(aat);
        if (rc == ORC_OK) {
            double* btb = mm(Bt, n, q, B, n);
            double* z = right_solve_sym(w, m, n, btb, &rc, err);
            free(btb);
            if (rc == ORC_OK) {
                double* atz = mm(At, p, m, z, n);
                xs = mm(atz, p, n, Bt, q);
                free(atz);
            }
            free(z);
        }
        free(w);
        if (kind) *kind = ORC_REF_LEAST_NORM_FULL_ROW_COL;
    } else {
        double* Ap = (double*)malloc(sizeof(double) * p * m);
        double* Bp = (double*)malloc(sizeof(double) * n * q);
        rc = orc_pseudoinverse(A, m, p, rank_tol, Ap, err);
        if (rc == ORC_OK) rc = orc_pseudoinverse(B, q, n, rank_tol, Bp, err);
        if (rc == ORC_OK) {
            double* apc = mm(Ap, p, m, C, n);
            xs = mm(apc, p, n, Bp, q);
            free(apc);
        }
        free(Ap); free(Bp);
        if (kind) *kind = ORC_REF_LEAST_NORM_GENERAL;
    }
    free(At); free(Bt);
    if (rc != ORC_OK) {
        free(xs);
        return rc;
    }
    /* residual_check = frobenius_dist(A·X*·B, C) (analysis.hpp:86-90) */
    double* ax = mm(A, m, p, xs, q);
    double* axb = mm(ax, m, q, B, n);
    free(ax);
    double d = 0.0;
    for (size_t i = 0; i < m * n; ++i) {
        double t = axb[i] - C[i];
        d += t * t;
    }
    free(axb);
    d = sqrt(d);
    memcpy(X, xs, sizeof(double) * p * q);
    free(xs);
    if (residual_check) *residual_check = d;
    if (d > 1e-8 * (1.0 + sqrt(orc_frobenius_sq(C, m * n)))) {
        if (err) snprintf(err, 256, "reference_solution: system is not consistent (residual %f)", d);
        return ORC_DOMAIN_ERROR;
    }
    return ORC_OK;
}

int orc_bk_limit(const double* A, size_t m, size_t p, const double* B, size_t q, size_t n,
                 const double* C, const double* X0, double* out, char* err) {
    if (!m || !p || !q || !n) return set_err(err, ORC_SHAPE_ERROR, "svd: empty matrix");
    double* Ap = (double*)malloc(sizeof(double) * p * m);
    double* Bp = (double*)malloc(sizeof(double) * n * q);
    int rc = orc_pseudoinverse(A, m, p, -1.0, Ap, err);
    if (rc == ORC_OK) rc = orc_pseudoinverse(B, q, n, -1.0, Bp, err);
    if (rc == ORC_OK) {
        double* apc = mm(Ap, p, m, C, n);
        double* xs = mm(apc, p, n, Bp, q);
        double* ax = mm(A, m, p, X0, q);
        double* axb = mm(ax, m, q, B, n);
        double* t = mm(Ap, p, m, axb, n);
        double* proj = mm(t, p, n, Bp, q);
        for (size_t i = 0; i < p * q; ++i) out[i] = xs[i] + (X0[i] - proj[i]);
        free(apc); free(xs); free(ax); free(axb); free(t); free(proj);
    }
    free(Ap); free(Bp);
    return rc;
}

int orc_rrn(const double* xk, const double* ref, size_t len, double* out, char* err) {
    const double ref_sq = orc_frobenius_sq(ref, len);
    if (ref_sq == 0.0) return set_err(err, ORC_DOMAIN_ERROR, "rrn: zero reference");
    double d = 0.0;
    for (size_t i = 0; i < len; ++i) {
        double t = xk[i] - ref[i];
        d += t * t;
    }
    *out = d / ref_sq;
    return ORC_OK;
}
