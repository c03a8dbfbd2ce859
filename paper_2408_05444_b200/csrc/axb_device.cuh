// axb_device.cuh — device-side state and kernel interfaces of the B200 solver.
//
// The reference keeps the whole iteration state in host memory inside
// axb::Solver (solver.hpp:496-514).  Here it lives in HBM: the matrices in
// row-major FP64 buffers and the scalar state (iteration counter, xoshiro256**
// stream, selected row, running reductions, stop flags) in one DevState block
// that every kernel of an iteration reads, so an iteration needs no host
// round trip and a batch of iterations is one captured CUDA graph.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace axb_dev {

// status values of DevState::status
enum : int32_t {
    ST_RUN = 0,       // iterate
    ST_PAUSE = 1,     // tracked stop metric <= tol: host confirms (solver.hpp:351-358)
    ST_ZERO = 2,      // ‖R‖² == 0 in run(): nothing to select (solver.hpp:347)
    ST_ERROR = 3      // err_code holds the axb_status (DivergenceError, DomainError, …)
};

// finalize modes of the residual kernel
enum : int32_t {
    FIN_NORMS = 0,     // init / adopt: norms + reductions + (re)select
    FIN_ITERATION = 1, // a step(): k++, trace, stop check, pre-select the next row
    FIN_UPDATE_ROW = 2 // public update_row(i): no k++, no trace, no stop check
};

struct alignas(16) DevState {
    // control
    unsigned long long k;        // iterations completed
    unsigned long long k_limit;  // kernels are no-ops once k >= k_limit
    unsigned long long k0;       // iteration index stored in trace slot 0
    int32_t status;
    int32_t err_code;
    unsigned long long err_k;
    double err_val;
    int32_t fin_mode;
    int32_t run_mode;            // 1 inside run() (zero-residual break), 0 in step()/steps()
    // selection (rng.hpp:18-123 state; solver.hpp:511 cyclic_pos_, skipped_zero_rows_)
    unsigned long long rng[4];
    unsigned long long cyclic_pos;
    unsigned long long skipped_zero_rows;
    // snapshot taken before the speculative pre-selection (rolled back when R
    // changes outside the iteration pipeline or a public select_* is called)
    unsigned long long rng_snap[4];
    unsigned long long cyclic_snap;
    unsigned long long skipped_snap;
    int32_t sel_valid;
    int32_t tie_guard_hits;
    long long sel;               // selected row (global index)
    double coef;                 // α / ‖A_sel‖²
    // reductions of the current residual
    double r_fro_sq;             // Σ_l ‖R_l‖² (fresh tree sum)
    double max_ratio;            // max_l ‖R_l‖²/‖A_l‖²
    long long argmax;            // smallest l attaining it
    double err_sq;               // ‖X − X_ref‖²_F (fresh, solution_rrn)
    double metric;               // current stop metric
    int32_t x_finite;            // X all finite (checkpoint guard, solver.hpp:428)
    int32_t sel_pending;         // K2 left the greedy pre-selection to k_sel_greedy
    // query results (greedy_threshold / max_residual_ratio)
    double q_zeta;
    long long q_row;
    long long q_count;
    // self-resetting last-block counters
    unsigned int cnt_r;
    unsigned int cnt_x;
    unsigned int cnt_red;
    unsigned int cnt_sel;        // k_sel_greedy last-block counter
    unsigned long long r_next;   // dynamic row counter of the TMA residual kernel
    int32_t replay;              // 1: select from Params::forced_rows (index-stream replay)
    int32_t packed;              // sharded: this rank's pack_send holds the last row
    int32_t pack_prev;           // sharded: ... held the row before (k_pack clears it)
    unsigned int cnt_sel1;       // k_sel1 last-block counter
    unsigned int cnt_yg;         // k_yg_tma last-block counter
    unsigned long long yg_next;  // dynamic row counter of k_yg_tma
    unsigned long long dbg[8];   // phase timestamps of the last greedy selection (ns)
};

struct RowRecord {   // per-CTA partial of the residual reduction
    double sum;      // Σ ‖R_l‖² over the CTA's rows
    double max_ratio;
    long long argmax;
    double _pad;
};

// Everything an iteration needs; constant for the life of a solver, so the
// captured graph's kernel parameters never change.
struct Params {
    long long m, p, q, n;        // m = local rows of A, C, R
    long long row0;              // global index of local row 0
    long long m_global;
    const double* A;             // m×p
    const double* B;             // q×n
    double* R;                   // m×n
    double* X;                   // p×q
    const double* Xref;          // p×q or null
    const double* a_sq;          // m   (host-computed in reference order)
    const double* rbk_cum;       // m_global (host-computed in reference order)
    double* r_sq;                // m
    const double* G;             // cached Gram columns: G[i*m + l] = A_i·A_l, or null
    double* g;                   // m   (when G is null)
    double* y;                   // q
    double* z;                   // n
    double* zpart;               // nzj × n
    unsigned int* zcnt;          // nslab counters
    double* xpart;               // x-update partials
    RowRecord* rrec;             // residual partials
    long long* trace_row;        // batch trace of selected rows
    double* trace_metric;        // batch trace of the stop metric
    double* trace_rel;           // batch trace of ‖R‖/‖C‖
    unsigned long long trace_cap;
    int* member_flags;           // m (greedy_index_set query)
    const long long* forced_rows;  // replayed index stream, slot = k − k0
    double* gsum;                // ⌈m/32⌉ group member masses (selection scratch)
    // ---- row sharding over `world` ranks (pack == nullptr: single GPU) ----
    int world, rank;
    double* pack;                // n + p + 2 (allreduced): R_i | A_i | sel | coef
    double* pack_send;           // this rank's contribution (zeros unless owner)
    double* recs;                // world × 4 (allgathered): Σ‖R_l‖², max ratio, argmax, err
    double* r_sq_g;              // m_global ‖R_l‖² (allgathered; r_sq points at this rank's slice)
    const double* a_sq_g;        // m_global ‖A_i‖² (allgathered), for BK/RBK/replay
    long long c0, c1;            // this rank's column slice of B for y and z
    long long x0r, x1r;          // this rank's rows of X
    DevState* st;
    double alpha, theta, a_fro_sq, tol, ref_sq, c_fro;
    int method, stop_kind, tie_guard, vec2;
    // launch geometry
    int r_grid, r_rows_per_cta, r_chunk, r_tma, r_stages, r_zstage;
    int r_grab;  // K2 producer: rows taken per atomic grab (1..32)
    int persist, persist_grid;   // small systems: one cooperative kernel per batch
    int persist_lat;             // latency body (threads per CTA, 0 = off): selection state in
                                 // shared memory, 2 barriers per iteration (m ≤ kPersistLatRows)
    const double* BtB;           // n×n BᵀB (solver.hpp:172) for z = BᵀB·R_iᵀ in one phase, or null
    int yg_grid, yg_rbq, yg_rbm;  // K4 grid; B rows / A rows per CTA
    int yg_tma;                  // K4 as a TMA ring (k_yg_tma) instead of k_yg
    int yg_pf;                   // K4: bytes of its first B rows a CTA prefetches into L2
                                 // before the selection it depends on has finished (0 = off)
    int sel_early;               // K3 lets K4 launch (and prefetch) before K2 has drained
    int z_nslab, z_nj, z_jrows, x_ctas;
    int sel1_grid, pack_grid;  // sharded selection: membership CTAs, row-pack CTAs
    int sel_split, sel_grid;     // greedy pre-selection across sel_grid CTAs (k_sel_greedy)
    // ---- CSR operands (null = dense).  The persistent general body
    // iterates stored entries only, as the reference's Solver<SparseMatrix,…> does
    // (solver.hpp:272-273, 294-295, 489-492): y = B·R_iᵀ over B's rows, z = yᵀ·B over
    // Bᵀ's rows (B's columns), the X update over A_i's entries, the R update over
    // the CSR Gram row G_i (scattered into g, zero elsewhere) ----
    const long long* a_rp; const int* a_ci; const double* a_v;     // A  m×p
    const long long* g_rp; const int* g_ci; const double* g_v;     // G = A·Aᵀ (m×m)
    const long long* b_rp; const int* b_ci; const double* b_v;     // B  q×n
    const long long* bt_rp; const int* bt_ci; const double* bt_v;  // Bᵀ n×q
    const long long* btb_rp; const int* btb_ci; const double* btb_v;  // BᵀB n×n (latency body)
};

// ---- checked build (-DAXB_CHECKED, libaxb_b200_checked.so) ----
// compute-sanitizer is not available on the GPU pool, so the checked build
// carries its own bounds checks at the iteration kernels' indexing sites: the
// first violated check records its source line in a device word (no trap: the
// context stays usable) and the host raises AXB_CUDA_ERROR at its next state
// pull.  The production build compiles the checks out.
#ifdef AXB_CHECKED
// the flag word g_axb_violation is defined in axb_iter.cu, the checks' only TU
#define AXB_CHECK(c)                                                                    \
    do {                                                                                \
        if (!(c)) atomicCAS(&axb_dev::g_axb_violation, 0ull, (unsigned long long)__LINE__); \
    } while (0)
#else
#define AXB_CHECK(c) ((void)0)
#endif
// 0, or the axb_iter.cu line of the first failed check since the last call (then cleared)
unsigned long long checked_violation();

// ---- launchers (axb_iter.cu) ----
void launch_yg(const Params& P, cudaStream_t s, bool with_g);
void launch_zx(const Params& P, cudaStream_t s);
void launch_r(const Params& P, cudaStream_t s, bool update);
// greedy pre-selection of the next row after K2 when P.sel_split (PDL-chained)
void launch_sel_greedy(const Params& P, cudaStream_t s);
void launch_select(const Params& P, cudaStream_t s, int method, double theta, int consume);
void launch_query(const Params& P, cudaStream_t s, double theta, int want_set);
void launch_rollback(const Params& P, cudaStream_t s);
void launch_err_fresh(const Params& P, cudaStream_t s);
// T = S·X for a CSR S (rows × p) and dense X (p × q), row-major T (rows × q):
// T_i = Σ_e S_v[e]·X[S_ci[e], :] over S_i's stored entries in order
// (matrix.hpp sparse matmul), one warp per row
void launch_spmm_csr(const long long* rp, const int* ci, const double* v, long long rows,
                     const double* X, long long q, double* T, cudaStream_t s);
// device power iteration helpers: y = M v (rows), w = Mᵀ y (cols)
void launch_rowdot(const double* M, long long rows, long long cols, const double* v, double* out,
                   cudaStream_t s);
void launch_coldot(const double* M, long long rows, long long cols, const double* v, double* out,
                   double* part, unsigned int* cnt, int nj, int jrows, cudaStream_t s);
void launch_power_step(const double* v_in, const double* w, double* v_out, long long dim,
                       double* out2, cudaStream_t s);
void launch_fill(double* p, long long n, double v, cudaStream_t s);
constexpr int kZxWarps = 8;  // warps per k_zx CTA (X rows per CTA)
void launch_power_step2(double* v, const double* w, long long dim, double* ps, double tol,
                        double max_iter, cudaStream_t s);
void launch_transpose(const double* in, long long rows, long long cols, double* out,
                      cudaStream_t s);
void launch_ctrl(DevState* st, unsigned long long k0, unsigned long long k_limit, int fin_mode,
                 int run_mode, int reset_status, cudaStream_t s);
void launch_set_sel(DevState* st, long long sel, double coef, cudaStream_t s);
void launch_set_replay(DevState* st, int on, cudaStream_t s);
int sumsq_parts(long long n);
void launch_sumsq(const double* v, long long n, double* part, cudaStream_t s);
void launch_row_sq_seq(const double* A, long long m, long long p, double* out, cudaStream_t s);
void launch_cumsum_seq(const double* a_sq, long long m, double* cum, double* total, cudaStream_t s);
// sharded selection (between the r_sq / record allgather and the row allreduce):
// mode 0 norms only, 1 iteration (+ select, + k_pack), 2 select only (+ k_pack)
void launch_sel1(const Params& P, cudaStream_t s, int mode);
// persistent cooperative batch kernel for small systems; returns a cudaError_t
int launch_persist(const Params& P, cudaStream_t s);
// many independent small systems, one CTA each (dPs: device array of Params)
int launch_persist_batch(const Params* dPs, int count, long long max_m, cudaStream_t s);
// rows up to which the latency body runs (every CTA re-reads r_sq each iteration and
// selects from shared memory; above this the per-CTA records of the general body win)
constexpr long long kPersistLatRows = 2048;

// ---- DMMA GEMM (axb_gemm.cu) ----
// D = (Cin ? Cin − A·op(B) : A·op(B)); op(B) = B (K×N) or Bᵀ (B is N×K) when b_trans.
// Optional per-CTA partials: sum of D² (sq_part) and of (Rold − D)² (diff_part),
// reduced deterministically by reduce_parts().  store=0 skips writing D.
struct GemmArgs {
    long long M, N, K;
    const double* A; long long lda;
    const double* B; long long ldb;
    int b_trans;
    double* D; long long ldd;
    const double* Cin; long long ldc;
    const double* Rold; long long ldr;
    double* sq_part;
    double* diff_part;
    int store;
    int sym;  // D = A·Aᵀ: compute only tiles on/above the diagonal (mirror with launch_mirror_lower)
    int no_pf;  // k_dgemm_tma: skip the L2 prefetch of the epilogue operands (AXB_GEMM_PF=0)
};
int timeline_read(unsigned long long* out, int reset);
int gemm_num_ctas(long long M, long long N);
void launch_gemm(const GemmArgs& g, cudaStream_t s);
void launch_reduce_parts(const double* part, long long n, double* out, cudaStream_t s);
// D[i][j] = D[j][i] for the strictly-lower 32×32 blocks of a square matrix
void launch_mirror_lower(double* D, long long nn, long long ld, cudaStream_t s);

}  // namespace axb_dev
