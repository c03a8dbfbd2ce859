/*
 * axb_oracle.h — CPU ORACLE (test infrastructure only).
 *
 * A plain-C restatement of the reference solver path of arXiv 2408.05444's
 * implementation (`proj/include/axb/{solver,rng,matrix,decomp}.hpp`).  It is the
 * checker the CUDA product is compared against; it is NEVER linked into, called
 * by, or shipped with the product.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pin: the restatement is compiled with -ffp-contract=off and follows the
 * reference's loop orders, so on the same inputs it is BITWISE equal to the
 * reference `axb::Solver` (checked by tests/test_oracle.py against
 * oracle/_ref/libaxbref.so, a driver compiled directly from the reference headers,
 * and against the committed golden vectors in tests/golden/ made by that driver).
 */
#ifndef AXB_ORACLE_H
#define AXB_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes == product C-ABI codes == reference exception types (errors.hpp:10-72). */
enum {
    ORC_OK = 0,
    ORC_SHAPE_ERROR = 1,       /* axb::ShapeError */
    ORC_DOMAIN_ERROR = 2,      /* axb::DomainError */
    ORC_CONFIG_ERROR = 3,      /* axb::ConfigError */
    ORC_DIVERGENCE_ERROR = 4,  /* axb::DivergenceError{iteration,residual_norm} */
    ORC_INVARIANT_ERROR = 5,   /* axb::InvariantError */
    ORC_CONVERGENCE_ERROR = 6, /* axb::ConvergenceError{last_estimate} */
    ORC_DECOMPOSITION_ERROR = 9 /* axb::DecompositionError (errors.hpp:48-50) */
};

/* MethodTag (solver.hpp:16), AlphaRule (:68), StopRule::Kind (:80). */
enum { ORC_BK = 0, ORC_RBK = 1, ORC_GRBK = 2, ORC_RGRBK = 3, ORC_MWRBK = 4 };
enum { ORC_ALPHA_SAFE = 0, ORC_ALPHA_PAPER = 1, ORC_ALPHA_FIXED = 2 };
enum { ORC_STOP_SOLUTION_RRN = 0, ORC_STOP_RESIDUAL_REL = 1 };

/* SolveConfig (solver.hpp:100-109), flattened. */
typedef struct {
    int32_t method;
    int32_t has_theta;
    double theta;
    int32_t alpha_rule;
    int32_t stop_kind;
    double alpha_value;
    double tol;
    const double* reference; /* p×q row-major, SolutionRrn only (may be NULL) */
    uint64_t max_iter;
    uint64_t seed;
    int32_t record_trace;
    int32_t _pad;
    uint64_t refresh_interval;
} orc_config;

/* RngStream (rng.hpp:18-123). */
typedef struct {
    uint64_t s[4];
    uint64_t seed;
    double spare;
    int32_t has_spare;
} orc_rng;

void orc_rng_init(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next_u64(orc_rng* r);
double orc_rng_next_unit(orc_rng* r);
double orc_rng_gauss(orc_rng* r);
void orc_rng_substream(const orc_rng* r, uint64_t t, orc_rng* out);
/* returns index; *status = ORC_DOMAIN_ERROR when cum.back() <= 0 */
size_t orc_rng_categorical_cdf(orc_rng* r, const double* cum, size_t n, int* status);
void orc_dense_gaussian(orc_rng* r, size_t rows, size_t cols, double* out);

/* matrix.hpp primitives (dense, row-major). */
void orc_matmul(const double* a, size_t ar, size_t ac, const double* b, size_t bc, double* c);
void orc_gram_mmt(const double* a, size_t rows, size_t cols, double* g);
double orc_frobenius_sq(const double* a, size_t len);
double orc_spectral_norm(const double* mat, size_t rows, size_t cols, double tol,
                         size_t max_iter, int* status, double* last_estimate);

/* problems.hpp:345-364 generate() for two Gaussian sources: A m×p, B q×n, X* p×q,
 * C = (A·X*)·B.  Any output pointer may be NULL except those needed for C. */
void orc_generate_gaussian(uint64_t seed, size_t m, size_t p, size_t q, size_t n,
                           double* A, double* B, double* X, double* C);

/* ---- Solver<DenseMatrix,DenseMatrix> (solver.hpp:143-515) ---- */
typedef struct orc_solver orc_solver;

orc_solver* orc_solver_create(const double* A, size_t m, size_t p, const double* B, size_t q,
                              size_t n, const double* C, const double* X0,
                              const orc_config* cfg, int* status, char* errbuf, size_t errlen);
void orc_solver_destroy(orc_solver* s);
const char* orc_solver_last_error(const orc_solver* s);

int orc_solver_step(orc_solver* s, uint64_t* row);
int orc_solver_update_row(orc_solver* s, uint64_t i);
int orc_solver_select_cyclic(orc_solver* s, uint64_t* row);
int orc_solver_select_rbk(orc_solver* s, uint64_t* row);
int orc_solver_select_greedy(orc_solver* s, double theta, uint64_t* row);
int orc_solver_select_mwrbk(orc_solver* s, uint64_t* row);
int orc_solver_greedy_threshold(orc_solver* s, double theta, double* out);
int orc_solver_rgrbk_threshold(orc_solver* s, double theta, double* out);
/* members written to out (capacity m), count to *count */
int orc_solver_greedy_index_set(orc_solver* s, double theta, uint64_t* out, uint64_t* count);
int orc_solver_max_residual_ratio(orc_solver* s, uint64_t* row, double* ratio);
int orc_solver_checkpoint(orc_solver* s);
int orc_solver_exact_metric(orc_solver* s, double* out);
int orc_solver_exact_residual_rel(orc_solver* s, double* out);
int orc_solver_residual_drift(orc_solver* s, double* out);
double orc_solver_current_metric(const orc_solver* s);
double orc_solver_current_residual_rel(const orc_solver* s);

/* SolveReport (solver.hpp:120-133) minus the owned vectors. */
typedef struct {
    uint64_t iterations;
    double wall_seconds;
    double final_rrn;
    double final_residual_rel;
    int32_t terminated_by; /* 0 Tolerance, 1 MaxIter */
    int32_t alpha_outside_bound;
    double alpha;
    uint64_t seed;
    uint64_t skipped_zero_rows;
    uint64_t trace_len;
    uint64_t diverged_iteration;  /* DivergenceError payload */
    double diverged_residual;
} orc_report;

/* run() (solver.hpp:337-372).  Trace arrays (k, rrn, residual_rel, row) may be
 * NULL; when given they must have trace_cap entries (excess points are counted
 * in trace_len but not written).  X is copied out to x_out when non-NULL. */
int orc_solver_run(orc_solver* s, orc_report* rep, uint64_t* trace_k, double* trace_rrn,
                   double* trace_rel, uint64_t* trace_row, uint64_t trace_cap, double* x_out);

/* benchmark-only prepared state: caches borrowed from the caller (see .c) */
orc_solver* orc_solver_create_prepared(const double* A, size_t m, size_t p, const double* B,
                                       size_t q, size_t n, const double* C, const double* X0,
                                       const double* R0, const double* G, const double* BtB,
                                       double alpha, const orc_config* cfg, int* status);
int orc_solver_steps(orc_solver* s, uint64_t k, uint64_t* rows);

/* accessors (solver.hpp:376-385) */
uint64_t orc_solver_iteration(const orc_solver* s);
double orc_solver_alpha(const orc_solver* s);
double orc_solver_spectral_norm_b(const orc_solver* s);
int orc_solver_alpha_outside_bound(const orc_solver* s);
double orc_solver_a_fro_sq(const orc_solver* s);
double orc_solver_residual_fro_sq(const orc_solver* s);
void orc_solver_get_X(const orc_solver* s, double* out);
void orc_solver_get_R(const orc_solver* s, double* out);
void orc_solver_get_r_sq(const orc_solver* s, double* out);
void orc_solver_get_a_sq(const orc_solver* s, double* out);
void orc_solver_rng_state(const orc_solver* s, uint64_t out[4]);

/* ------------------------------------------------------------------------
 * Reference solutions: decomp.hpp svd / pseudoinverse / lu_solve
 * and analysis.hpp reference_solution / bk_limit / rrn, dense operands.
 * Errors: ORC_SHAPE_ERROR, ORC_DOMAIN_ERROR, ORC_DECOMPOSITION_ERROR; the
 * message is copied to err (≥ 256 bytes) when err is non-NULL.
 * ------------------------------------------------------------------------ */
enum { ORC_REF_UNIQUE_FULL_RANK = 0, ORC_REF_LEAST_NORM_FULL_ROW_COL = 1,
       ORC_REF_LEAST_NORM_GENERAL = 2 }; /* ReferenceCase (analysis.hpp:18) */

/* svd(M, max_sweeps) (decomp.hpp:113-157): r = min(rows, cols); U rows×r,
 * sigma r (nonincreasing), V cols×r, all row-major; any output may be NULL. */
int orc_svd(const double* M, size_t rows, size_t cols, size_t max_sweeps, double* U,
            double* sigma, double* V, size_t* numeric_rank, char* err);
/* pseudoinverse(M, rank_tol) (decomp.hpp:161-177): P is cols×rows. */
int orc_pseudoinverse(const double* M, size_t rows, size_t cols, double rank_tol, double* P,
                      char* err);
/* lu_solve(a, b) (decomp.hpp:249-279): a n×n, b n×k, both overwritten; b = a⁻¹b. */
int orc_lu_solve(double* a, size_t n, double* b, size_t k, char* err);
/* reference_solution(A, B, C, rank_tol) (analysis.hpp:48-91): X p×q. */
int orc_reference_solution(const double* A, size_t m, size_t p, const double* B, size_t q,
                           size_t n, const double* C, double rank_tol, double* X, int* kind,
                           double* residual_check, char* err);
/* bk_limit(A, B, C, X0) (analysis.hpp:95-104): out p×q. */
int orc_bk_limit(const double* A, size_t m, size_t p, const double* B, size_t q, size_t n,
                 const double* C, const double* X0, double* out, char* err);
/* rrn(xk, reference) (analysis.hpp:107-111). */
int orc_rrn(const double* xk, const double* ref, size_t len, double* out, char* err);

#ifdef __cplusplus
}
#endif
#endif
