/*
 * axb_b200.h — C-ABI of the B200-native row-action solver for A·X·B = C.
 *
 * Drop-in boundary for the reference's header-only engine
 * (/root/reference/proj/include/axb/solver.hpp).  Every entry point below names
 * the reference interface it replaces.  Plain pointers and sizes only; no torch
 * or CUDA types in the signatures.  All matrices are dense, row-major FP64
 * (matrix.hpp:37-70): A is m×p, B is q×n, C and R are m×n, X is p×q.
 *
 * Errors: every function returns an axb_status; the codes map 1:1 onto the
 * reference's exception types (errors.hpp:10-72).  The message of the last
 * failure on a handle is available from axb_solver_last_error().  The C++ shim
 * include/axb_b200/solver.hpp rethrows them as the axb:: exception types.
 *
 * Threading: a handle is single-owner and not thread-safe, like axb::Solver
 * (rng.hpp:15-17); different handles may run concurrently on
 * different devices/streams.  Every call on a handle runs on the handle's device
 * (axb_options.device) whatever the calling thread's current device is, and
 * leaves the caller's current device unchanged.
 *
 * There is no CPU fallback: creating a solver without a usable sm_100 device
 * fails with AXB_CUDA_ERROR.
 */
#ifndef AXB_B200_H
#define AXB_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AXB_B200_ABI_VERSION 1

typedef enum {
    AXB_OK = 0,
    AXB_SHAPE_ERROR = 1,       /* axb::ShapeError       errors.hpp:15-17 */
    AXB_DOMAIN_ERROR = 2,      /* axb::DomainError      errors.hpp:20-22 */
    AXB_CONFIG_ERROR = 3,      /* axb::ConfigError      errors.hpp:30-32 */
    AXB_DIVERGENCE_ERROR = 4,  /* axb::DivergenceError  errors.hpp:60-67 */
    AXB_INVARIANT_ERROR = 5,   /* axb::InvariantError   errors.hpp:70-72 */
    AXB_CONVERGENCE_ERROR = 6, /* axb::ConvergenceError errors.hpp:53-57 */
    AXB_CUDA_ERROR = 7,        /* device / runtime failure (no reference analogue) */
    AXB_CAPACITY_ERROR = 8,    /* axb::CapacityError    errors.hpp:25-27 (HBM exhausted) */
    AXB_DECOMPOSITION_ERROR = 9 /* axb::DecompositionError errors.hpp:48-50 */
} axb_status;

/* MethodTag (solver.hpp:16) */
enum { AXB_BK = 0, AXB_RBK = 1, AXB_GRBK = 2, AXB_RGRBK = 3, AXB_MWRBK = 4 };
/* AlphaRule (solver.hpp:68) */
enum { AXB_ALPHA_SAFE = 0, AXB_ALPHA_PAPER = 1, AXB_ALPHA_FIXED = 2 };
/* StopRule::Kind (solver.hpp:80) */
enum { AXB_STOP_SOLUTION_RRN = 0, AXB_STOP_RESIDUAL_REL = 1 };
/* Terminated (solver.hpp:118) */
enum { AXB_TERMINATED_TOLERANCE = 0, AXB_TERMINATED_MAX_ITER = 1 };

/* SolveConfig (solver.hpp:100-109), flattened.  `reference` is the p×q X_ref of
 * StopRule::solution_rrn (host pointer; copied at create). */
typedef struct {
    int32_t method;
    int32_t has_theta;
    double theta;
    int32_t alpha_rule;
    int32_t stop_kind;
    double alpha_value;
    double tol;
    const double* reference;
    uint64_t max_iter;
    uint64_t seed;
    int32_t record_trace;
    int32_t _pad;
    uint64_t refresh_interval;
} axb_config;

/* SolveReport (solver.hpp:120-133) minus the owned vectors (trace and X are
 * copied into caller buffers by axb_solver_run). */
typedef struct {
    uint64_t iterations;
    double wall_seconds;
    double final_rrn;
    double final_residual_rel;
    int32_t terminated_by;
    int32_t alpha_outside_bound;
    double alpha;
    uint64_t seed;
    uint64_t skipped_zero_rows;
    uint64_t trace_len;
    uint64_t diverged_iteration; /* DivergenceError::iteration */
    double diverged_residual;    /* DivergenceError::residual_norm */
} axb_report;

/* B200 placement / execution options (no reference analogue).  Zero-initialise
 * and set what you need; axb_options_default() fills the defaults. */
typedef struct {
    int32_t device;            /* CUDA ordinal */
    int32_t inputs_on_device;  /* 1: A,B,C,X0 (and cfg.reference) are device pointers */
    int32_t cache_gram;        /* -1 auto (fits in HBM and max_iter repays forming it),
                                  0 form g = A·A_iᵀ per step, 1 cache G = A·Aᵀ */
    int32_t spectral_on_device;/* -1 auto, 0 host (bitwise reference α), 1 device */
    int32_t graph_iters;       /* iterations captured per CUDA graph (0 = default) */
    int32_t tie_guard;         /* 1 (default): exact sequential re-check of near-boundary draws;
                                  0 off; 2 every greedy draw takes the sequential walk (test hook) */
    uint64_t spectral_max_iter;/* power-iteration cap (0 = reference default 5000) */
    double alpha_override;     /* >0: use this α verbatim (e.g. the oracle's), skip ‖B‖₂ */
    /* row sharding (§8(e)): this handle owns rows [row_offset, row_offset+m) of an
     * m_global-row system; NULL comm = single GPU. */
    void* nccl_comm;           /* ncclComm_t, or NULL */
    int32_t world_size;
    int32_t rank;
    uint64_t m_global;
    uint64_t row_offset;
    /* SMs this handle's persistent kernel (small systems) may occupy, 0 = all: set
     * it to share one GPU between handles that run concurrently on their own host
     * threads (e.g. config 4's colour channels: three handles at SMs/3 each). */
    int32_t sm_share;
    int32_t _pad0;
} axb_options;

typedef struct axb_solver axb_solver;

void axb_options_default(axb_options* opt);

/* ---- row sharding (§8(e)): NCCL bootstrap, one communicator per GPU/process ----
 * Rank 0 creates an id, the caller distributes it (e.g. torch.distributed
 * broadcast over gloo), every rank creates its communicator and passes it in
 * axb_options.nccl_comm with world_size, rank, m_global = world·m and
 * row_offset = rank·m (equal contiguous row shards).  NCCL is loaded at run
 * time (dlopen "libnccl.so.2"); single-GPU use never touches it. */
int axb_nccl_unique_id(unsigned char out[128]);
int axb_nccl_comm_create(int nranks, const unsigned char id[128], int rank, int device,
                         void** comm);
int axb_nccl_comm_destroy(void* comm);
/* Test infrastructure: `world` communicators of an in-process emulation of the
 * collectives (ranks = host threads of this process, one solver handle each, all
 * on one device; every collective synchronises at a host barrier).  Lets the
 * row-sharded path run with world > 1 on a single GPU; destroy each with
 * axb_nccl_comm_destroy.  Not for performance: iterations are not graph-captured. */
int axb_nccl_emulated_group(int world, void** comms);
int axb_abi_version(void);
/* 1 in the bounds-checked build (libaxb_b200_checked.so, -DAXB_CHECKED): the
 * iteration kernels check their indexing and a violation fails the next call
 * with AXB_CUDA_ERROR ("device bounds check failed at axb_iter.cu:<line>"). */
int axb_checked_build(void);
/* 1 when a device that can run the sm_100a kernels is visible. */
int axb_device_available(void);

/* Solver::Solver(A, B, C, X0, cfg)  — solver.hpp:146-192.
 * A m×p, B q×n, C m×n, X0 p×q (NULL = zeros). */
int axb_solver_create(const double* A, uint64_t m, uint64_t p, const double* B, uint64_t q,
                      uint64_t n, const double* C, const double* X0, const axb_config* cfg,
                      const axb_options* opt, axb_solver** out);
void axb_solver_destroy(axb_solver* s);
const char* axb_solver_last_error(const axb_solver* s);
/* payload of the last DivergenceError (iteration, residual norm) or
 * ConvergenceError (last estimate in *value) raised on this handle */
int axb_solver_last_error_info(const axb_solver* s, uint64_t* iteration, double* value);
/* message for failures of axb_solver_create (handle-less), thread-local */
const char* axb_last_create_error(void);

/* Storage-agnostic matrix descriptor: the reference's axb::Matrix variant
 * (matrix.hpp:178, DenseMatrix or CSR SparseMatrix :94-175).  kind 0 = dense
 * row-major `dense`; kind 1 = CSR (row_ptr[rows+1], col_idx[nnz] ascending per
 * row, values[nnz]), validated like SparseMatrix::validate.  Host pointers. */
typedef struct {
    int32_t kind;
    int32_t _pad;
    uint64_t rows, cols, nnz;
    const double* dense;
    const uint64_t* row_ptr;
    const uint64_t* col_idx;
    const double* values;
} axb_matrix;

/* solve(const Matrix& A, const Matrix& B, …) dispatch — solver.hpp:518-526, i.e.
 * Solver<AMat,BMat> over dense or CSR operands.  CSR operands are validated as
 * SparseMatrix does (matrix.hpp:94-175: ascending columns, finite non-zero
 * values) and STAY SPARSE on the device: a CSR A is never expanded — its Gram
 * G = A·Aᵀ is formed as CSR in the reference's order (matrix.hpp:496-535) and the
 * iteration walks stored entries only (X over nz(A_i), R over nz(G_i),
 * solver.hpp:272-273, :294-295); a CSR B is kept as CSR together with Bᵀ for the
 * y and z passes (:489-492), plus one dense q×n copy for ‖B‖₂ and the residual
 * GEMM (the reference itself holds the dense n×n BᵀB, :172).  Host arrays only.
 * Row-sharded handles (opt.nccl_comm) take dense operands: CSR is expanded
 * there, every stored-entry loop then adding exact zeros. */
int axb_solver_create_ex(const axb_matrix* A, const axb_matrix* B, const double* C,
                         const double* X0, const axb_config* cfg, const axb_options* opt,
                         axb_solver** out);

/* Solver::step() — solver.hpp:321-333.  One iteration; returns the row. */
int axb_solver_step(axb_solver* s, uint64_t* row);
/* k consecutive step() calls (the acceptance.cpp:128-141 driver loop, batched
 * on the device).  rows (may be NULL) receives the k selected rows.  When
 * mirror_refresh is set, checkpoint() runs every cfg.refresh_interval
 * iterations exactly as run() schedules it (solver.hpp:359-360). */
int axb_solver_steps(axb_solver* s, uint64_t k, uint64_t* rows, int32_t mirror_refresh);
/* k iterations on a GIVEN index stream (e.g. the reference's, from its trace):
 * each step applies update_row(rows[t]) and advances k, the RNG draw / cyclic
 * position and the refresh schedule exactly as step() would, so a randomized
 * run can be replayed and its iterates compared (north star: "randomized
 * variants, replaying the reference's index stream").  A zero row of A yields
 * AXB_DOMAIN_ERROR as update_row does. */
int axb_solver_replay(axb_solver* s, uint64_t k, const uint64_t* rows, int32_t mirror_refresh);
/* Solver::update_row(i) — solver.hpp:264-318. */
int axb_solver_update_row(axb_solver* s, uint64_t i);
/* Solver::run() — solver.hpp:337-372.  trace_* (may be NULL) receive up to
 * trace_cap TracePoints (:111-116); x_out (may be NULL) receives X (p×q). */
int axb_solver_run(axb_solver* s, axb_report* rep, uint64_t* trace_k, double* trace_rrn,
                   double* trace_rel, uint64_t* trace_row, uint64_t trace_cap, double* x_out);

/* selection rules, as public methods of Solver (solver.hpp:197-258, 387-400) */
int axb_solver_select_cyclic(axb_solver* s, uint64_t* row);
int axb_solver_select_rbk(axb_solver* s, uint64_t* row);
int axb_solver_select_greedy(axb_solver* s, double theta, uint64_t* row);
int axb_solver_select_mwrbk(axb_solver* s, uint64_t* row);
int axb_solver_greedy_threshold(axb_solver* s, double theta, double* out);
int axb_solver_rgrbk_threshold(axb_solver* s, double theta, double* out);
int axb_solver_greedy_index_set(axb_solver* s, double theta, uint64_t* out, uint64_t* count);
int axb_solver_max_residual_ratio(axb_solver* s, uint64_t* row, double* ratio);

/* metrics and drift checkpoint (solver.hpp:403-436) */
int axb_solver_current_metric(axb_solver* s, double* out);
int axb_solver_current_residual_rel(axb_solver* s, double* out);
int axb_solver_exact_metric(axb_solver* s, double* out);
int axb_solver_exact_residual_rel(axb_solver* s, double* out);
int axb_solver_residual_drift(axb_solver* s, double* out);
int axb_solver_checkpoint(axb_solver* s);

/* accessors (solver.hpp:376-385); copy-out into caller-owned host buffers */
uint64_t axb_solver_iteration(const axb_solver* s);
double axb_solver_alpha(const axb_solver* s);
double axb_solver_spectral_norm_b(const axb_solver* s);
int axb_solver_alpha_outside_bound(const axb_solver* s);
/* 1 when G = A·Aᵀ is cached (axb_options.cache_gram), 0 when g = A·A_iᵀ is formed per step */
int axb_solver_gram_cached(const axb_solver* s);
double axb_solver_a_fro_sq(const axb_solver* s);
int axb_solver_residual_fro_sq(axb_solver* s, double* out);
int axb_solver_get_X(axb_solver* s, double* out);        /* p×q */
int axb_solver_get_R(axb_solver* s, double* out);        /* m×n (local rows) */
int axb_solver_get_r_sq(axb_solver* s, double* out);     /* m */
int axb_solver_get_a_sq(axb_solver* s, double* out);     /* m */
int axb_solver_dims(const axb_solver* s, uint64_t dims[4]); /* m, p, q, n */

/* ---- measurement hooks (bench.py) ---- */
/* run() on many independent handles of one device at once — the benchmark
 * pool's problem × method × trial sweep (analysis.hpp:255-356).
 * Small systems (those on the persistent-kernel path) advance together in ONE
 * launch per refresh segment, one CTA per system (k_persist_batch); larger ones
 * run their own launches in turn.  Each handle's result is exactly what
 * axb_solver_run would give: reps[i], x_outs[i] (may be NULL, or hold NULLs),
 * statuses[i] (its status code; message in axb_solver_last_error(hs[i])).
 * Returns AXB_OK unless the batch itself could not run. */
int axb_solvers_run(axb_solver* const* hs, uint32_t count, axb_report* reps,
                    double* const* x_outs, int32_t* statuses);
/* Device time (ms) of the last run()/steps() loop, CUDA events on the solver's
 * stream, and the summed device time of the residual-update kernel (K2) inside
 * it, with its launch count. */
int axb_solver_last_timing(const axb_solver* s, double* loop_ms, double* k2_ms,
                           uint64_t* k2_launches, uint64_t* kernel_launches);
/* Diagnostics: out[5] = greedy selections made, out[6] = exact sequential
 * fallbacks taken by the tie guard; out[0..4], out[7] = selection phase
 * timestamps (ns) when built with -DAXB_TRACE_SELECT. */
int axb_solver_debug_state(axb_solver* s, uint64_t out[8]);
/* Average per-launch device times (ms) of K4 (y), K4b+K5 (z, X) and K2 over the
 * last profiled steps()/run(), CUDA events between consecutive launches. */
int axb_solver_kernel_times(const axb_solver* s, double out_ms[3]);
/* Row-sharded solvers: average per-iteration device times (ms) of the exchange
 * steps over the last profiled steps()/run(): [0] y allreduce, [1] z allgather,
 * [2] the grouped ‖R_l‖²-slice + record allgather, [3] the global selection
 * kernels (k_sel1 + k_pack), [4] the selected-row allreduce.  Zeros on one GPU. */
int axb_solver_collective_times(const axb_solver* s, double out_ms[5]);
/* Diagnostics: the graph path's in-pipeline kernel timeline, a ring of 64
 * iterations × {K4, K4b+K5, K2, K3} × {earliest CTA start, latest CTA end} in
 * device-clock ns (out[64*8]); `reset` re-arms it.  Returns 1 when the library
 * was built with -DAXB_TRACE_TIMELINE, else 0 (out zeroed). */
int axb_debug_timeline(uint64_t out[512], int32_t reset);
/* Diagnostics: time K1 alone.  D = Cin − A·B (Cin may be NULL: D = A·B) on DEVICE
 * pointers, row-major FP64: A is M×K; B is K×N, or N×K when b_trans (D = A·Bᵀ).
 * Runs one untimed launch and `reps` timed ones on the current device; *ms is
 * the average device time of a launch (CUDA events). */
int axb_debug_dgemm(const double* A, const double* B, const double* Cin, double* D, uint64_t M,
                    uint64_t N, uint64_t K, int32_t b_trans, int32_t reps, double* ms);
/* Enable per-kernel CUDA-event timing of K2 inside steps()/run() (adds events to
 * the captured graph; off by default). */
int axb_solver_set_profiling(axb_solver* s, int32_t on);

/* ------------------------------------------------------------------------
 * Reference solutions on the device — the X* producers of
 * analysis.hpp / decomp.hpp, one-sided Jacobi in round-robin order plus DMMA
 * GEMMs (csrc/axb_analysis.cu).  Host pointers in and out, dense row-major;
 * `device` is the CUDA ordinal.  Failures return the status of the reference's
 * exception and leave the message in axb_last_create_error().
 * ------------------------------------------------------------------------ */
/* ReferenceCase (analysis.hpp:18) */
enum { AXB_REF_UNIQUE_FULL_RANK = 0, AXB_REF_LEAST_NORM_FULL_ROW_COL = 1,
       AXB_REF_LEAST_NORM_GENERAL = 2 };

/* svd(M, max_sweeps) — decomp.hpp:113-157.  r = min(rows, cols): sigma[r]
 * nonincreasing, U rows×r, V cols×r (any output may be NULL), numeric_rank at
 * the cutoff 8·max(rows,cols)·σ_max·2⁻⁵² (:30-33).  ShapeError on an empty M,
 * DecompositionError when max_sweeps sweeps do not converge. */
int axb_svd(const double* M, uint64_t rows, uint64_t cols, uint64_t max_sweeps, int32_t device,
            double* U, double* sigma, double* V, uint64_t* numeric_rank);
/* pseudoinverse(M, rank_tol) — decomp.hpp:161-177; P is cols×rows; rank_tol < 0
 * selects the default cutoff. */
int axb_pseudoinverse(const double* M, uint64_t rows, uint64_t cols, double rank_tol,
                      int32_t device, double* P);
/* reference_solution(A, B, C, rank_tol) — analysis.hpp:48-91: X p×q, kind one of
 * AXB_REF_*, residual_check = ‖A·X·B − C‖_F; DomainError when the residual
 * exceeds 1e-8·(1 + ‖C‖_F) (X is not written then). */
int axb_reference_solution(const axb_matrix* A, const axb_matrix* B, const double* C,
                           double rank_tol, int32_t device, double* X, int32_t* kind,
                           double* residual_check);
/* bk_limit(A, B, C, X0) — analysis.hpp:95-104: A⁺CB⁺ + X0 − A⁺AX0BB⁺, p×q. */
int axb_bk_limit(const axb_matrix* A, const axb_matrix* B, const double* C, const double* X0,
                 int32_t device, double* X);
/* rrn(Xk, reference) — analysis.hpp:107-111 (squared relative error). */
int axb_rrn(const double* Xk, const double* ref, uint64_t len, int32_t device, double* out);
/* Jacobi sweeps of the last call's factorisations on this thread (A, B) and its
 * device time in ms (CUDA events, inputs already resident). */
int axb_analysis_stats(uint64_t sweeps[2], double* device_ms);

#ifdef __cplusplus
}
#endif
#endif /* AXB_B200_H */
