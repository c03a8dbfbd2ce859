// axb_analysis.cu — reference solutions on the device.
//
// Replaces the host path the reference uses to produce X* for solution_rrn
// stopping and for the benchmark harness: analysis.hpp reference_solution
// (:48-91), bk_limit (:95-104) and rrn (:107-111), over decomp.hpp svd
// (:113-157) and pseudoinverse (:161-177).
//
// SVD.  The reference runs one-sided cyclic Jacobi (decomp.hpp:71-109): column
// pairs (p, q) in row-cyclic order, one at a time.  Here a sweep is ordered as
// a round-robin tournament: the N/2 pairs of a round are disjoint, so they
// rotate concurrently, one CTA per pair.  W is kept transposed (column j of W is
// row j of Wc, contiguous), so a pair is two coalesced streams: pass 1 forms
// app/aqq/apq with a fixed-order block reduction, pass 2 rotates the two W
// columns (re-read from L2) and the two V columns.  The rotation formula, the
// skip tests (null columns below ‖W‖²·1e-30, |apq| <= 1e-15·sqrt(app·aqq)), the
// "no rotation in a full sweep" stop and the 64-sweep cap are the reference's;
// the rotation ORDER differs, so factors agree with the reference to rounding,
// not bitwise (tests/test_gpu_analysis.py states the tolerances).
//
// Pseudoinverse.  With w_k = σ_k·u_k the Jacobi output gives
// A⁺ = Σ_{σ_k > tol} v_k w_kᵀ / σ_k², one DMMA GEMM (axb_gemm.cu) after scaling
// rows of the transposed factor — no U is ever normalised for A⁺.
//
// reference_solution.  The reference picks normal-equation LU solves for the two
// full-rank cases (:70-81) and pseudoinverses otherwise; all three are A⁺CB⁺ in
// exact arithmetic, so the device always evaluates (A⁺·C)·B⁺ on the GEMM (the SVD
// route is the better-conditioned one), inverting every positive σ in the
// full-rank cases as the LU solves do, and reports the reference's
// ReferenceCase label from the same rank tests.  The consistency guard
// (:86-90) is evaluated with the fused C − (A·X*)·B epilogue.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <new>
#include <numeric>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/axb_b200.h"
#include "axb_device.cuh"

namespace axb_dev {
std::string& handleless_error();
int expand_matrix(const axb_matrix* M, std::vector<double>& out, const char* name);
}  // namespace axb_dev

namespace axb_dev {
namespace {

constexpr int kJT = 256;              // threads per pair CTA
constexpr double kJacobiTol = 1e-15;  // decomp.hpp:73

// Round-robin ("circle") schedule over N (even) slots: in round r slot N−1
// meets r, and (r+k) meets (r−k) mod (N−1).  Every pair meets exactly once in
// rounds 0..N−2 and the pairs of one round are disjoint.
__device__ __forceinline__ void tournament_pair(int N, int round, int k, int& p, int& q) {
    int a, b;
    if (k == 0) {
        a = round;
        b = N - 1;
    } else {
        a = (round + k) % (N - 1);
        b = (round - k + (N - 1)) % (N - 1);
    }
    p = min(a, b);
    q = max(a, b);
}

// One round: CTA-strided loop over the round's pairs.  The grid is sized so the
// pairs in flight (16·m bytes each) fit in L2, so pass 2 re-reads its columns
// from L2 instead of HBM (one CTA per pair measured 2× W read traffic, ncu).
template <bool VEC>
__global__ void __launch_bounds__(kJT) k_jacobi_round(double* __restrict__ W, long long m,
                                                      double* __restrict__ V, long long n, int N,
                                                      int round, double null_sq, int* rotated) {
    __shared__ double red[3][kJT / 32];
    __shared__ double cs[2];
    __shared__ int go;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int k = blockIdx.x; k < N / 2; k += gridDim.x) {
        int p, q;
        tournament_pair(N, round, k, p, q);
        if (q >= n) continue;  // the bye of an odd column count (block-uniform)
        double* wp = W + (long long)p * m;
        double* wq = W + (long long)q * m;
        double app = 0.0, aqq = 0.0, apq = 0.0;
        if (VEC) {
            const double2* a2 = reinterpret_cast<const double2*>(wp);
            const double2* b2 = reinterpret_cast<const double2*>(wq);
            const long long m2 = m >> 1;
#pragma unroll 4
            for (long long i = threadIdx.x; i < m2; i += kJT) {
                const double2 x = a2[i], y = b2[i];
                app += x.x * x.x + x.y * x.y;
                aqq += y.x * y.x + y.y * y.y;
                apq += x.x * y.x + x.y * y.y;
            }
        } else {
#pragma unroll 4
            for (long long i = threadIdx.x; i < m; i += kJT) {
                const double x = wp[i], y = wq[i];
                app += x * x;
                aqq += y * y;
                apq += x * y;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            app += __shfl_xor_sync(0xffffffffu, app, o);
            aqq += __shfl_xor_sync(0xffffffffu, aqq, o);
            apq += __shfl_xor_sync(0xffffffffu, apq, o);
        }
        if (lane == 0) {
            red[0][warp] = app;
            red[1][warp] = aqq;
            red[2][warp] = apq;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double a = 0.0, b = 0.0, c2 = 0.0;
            for (int w = 0; w < kJT / 32; ++w) {
                a += red[0][w];
                b += red[1][w];
                c2 += red[2][w];
            }
            int g = 1;  // the reference's two `continue` tests, verbatim (NaN-faithful)
            if (a <= null_sq || b <= null_sq) g = 0;
            else if (fabs(c2) <= kJacobiTol * sqrt(a * b)) g = 0;
            double c = 1.0, s = 0.0;
            if (g) {
                const double zeta = (b - a) / (2.0 * c2);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                c = 1.0 / sqrt(1.0 + t * t);
                s = c * t;
                *rotated = 1;
            }
            cs[0] = c;
            cs[1] = s;
            go = g;
        }
        __syncthreads();
        if (!go) continue;
        const double c = cs[0], s = cs[1];
        if (VEC) {
            double2* a2 = reinterpret_cast<double2*>(wp);
            double2* b2 = reinterpret_cast<double2*>(wq);
            const long long m2 = m >> 1;
#pragma unroll 4
            for (long long i = threadIdx.x; i < m2; i += kJT) {
                const double2 x = a2[i], y = b2[i];
                a2[i] = make_double2(c * x.x - s * y.x, c * x.y - s * y.y);
                b2[i] = make_double2(s * x.x + c * y.x, s * x.y + c * y.y);
            }
        } else {
            for (long long i = threadIdx.x; i < m; i += kJT) {
                const double x = wp[i], y = wq[i];
                wp[i] = c * x - s * y;
                wq[i] = s * x + c * y;
            }
        }
        double* vp = V + (long long)p * n;
        double* vq = V + (long long)q * n;
        for (long long i = threadIdx.x; i < n; i += kJT) {
            const double x = vp[i], y = vq[i];
            vp[i] = c * x - s * y;
            vq[i] = s * x + c * y;
        }
    }
}

// CTAs per round: enough to fill the SMs, few enough that the columns of the
// pairs in flight mostly stay L2-resident between the two passes (≈ 96 MB of
// 126 MB; tools/sweep_jacobi.sh at config 3: 148 CTAs 123 µs/round, 296 83,
// 592 66, one per pair (1024) 72)
int jacobi_grid(long long m, long long n, int N) {
    int sms = 148;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (const char* e = std::getenv("AXB_JACOBI_CTAS")) return std::max(1, std::min(N / 2, std::atoi(e)));
    const long long per_pair = 16 * (m + n);
    const long long fit = std::max<long long>(sms, (96ll << 20) / std::max<long long>(per_pair, 1));
    return (int)std::max<long long>(1, std::min<long long>(N / 2, std::min<long long>(fit, 8ll * sms)));
}

__device__ double block_sum_fixed(double v) {
    __shared__ double red[kJT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    return t;  // valid in thread 0
}

// out[j] = ‖row j‖₂ — the column norms of W (decomp.hpp:119-124)
__global__ void __launch_bounds__(kJT) k_row_norms(const double* W, long long len, double* out) {
    const double* r = W + (long long)blockIdx.x * len;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < len; i += kJT) acc += r[i] * r[i];
    acc = block_sum_fixed(acc);
    if (threadIdx.x == 0) out[blockIdx.x] = sqrt(acc);
}

// dots[c] = U[c]·cand for c < j (classical Gram–Schmidt, first half)
__global__ void __launch_bounds__(kJT) k_gs_dots(const double* U, long long len,
                                                 const double* cand, double* dots) {
    const double* r = U + (long long)blockIdx.x * len;
    double acc = 0.0;
    for (long long i = threadIdx.x; i < len; i += kJT) acc += r[i] * cand[i];
    acc = block_sum_fixed(acc);
    if (threadIdx.x == 0) dots[blockIdx.x] = acc;
}

// cand −= Σ_{c<j} dots[c]·U[c] (second half)
__global__ void k_gs_sub(const double* U, long long len, int j, const double* dots, double* cand) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= len) return;
    double s = 0.0;
    for (int c = 0; c < j; ++c) s += dots[c] * U[(long long)c * len + i];
    cand[i] -= s;
}

__global__ void k_scale_rows(double* Y, long long rows, long long len, const double* d) {
    const long long total = rows * len;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x)
        Y[t] *= d[t / len];
}

// dst[j] = src[order[j]] / div[j] (div may be null) — sorted factor columns
__global__ void k_gather_rows(const double* src, long long len, const int* order,
                              const double* div, long long rows, double* dst) {
    const long long total = rows * len;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long j = t / len, i = t - j * len;
        const double v = src[(long long)order[j] * len + i];
        dst[t] = div ? v / div[j] : v;
    }
}

__global__ void k_set_diag(double* M, long long n, double v) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) M[i * n + i] = v;
}

__global__ void k_div_copy(const double* src, long long len, double d, double* dst) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < len) dst[i] = src[i] / d;
}

__global__ void k_add(const double* a, const double* b, long long n, double* out) {
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < n;
         t += (long long)gridDim.x * blockDim.x)
        out[t] = a[t] + b[t];
}

// parts of Σ (a − b)² and Σ b² (rrn, analysis.hpp:107-111)
__global__ void __launch_bounds__(kJT) k_rrn_parts(const double* a, const double* b, long long n,
                                                   double* part) {
    double d = 0.0, r = 0.0;
    for (long long t = (long long)blockIdx.x * kJT + threadIdx.x; t < n;
         t += (long long)gridDim.x * kJT) {
        const double x = a[t] - b[t];
        d += x * x;
        r += b[t] * b[t];
    }
    d = block_sum_fixed(d);
    __syncthreads();
    r = block_sum_fixed(r);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = d;
        part[gridDim.x + blockIdx.x] = r;
    }
}

int grid_for(long long n) {
    return (int)std::max<long long>(1, std::min<long long>(148 * 16, (n + 255) / 256));
}

// ---------------------------------------------------------------- host side

struct Fail {
    int code;
    std::string msg;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw Fail{code, buf};
}

void ck(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation)
        fail(AXB_CAPACITY_ERROR, "%s: out of device memory (%s)", what, cudaGetErrorString(e));
    fail(AXB_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
}

template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    Dev() = default;
    explicit Dev(size_t count) { alloc(count); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    Dev(Dev&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; }
    ~Dev() {
        if (p) cudaFree(p);
    }
    void alloc(size_t count) {
        if (p) cudaFree(p);
        p = nullptr;
        n = count;
        ck(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)), "cudaMalloc");
    }
};

struct Ctx {
    int prev = -1;
    cudaStream_t s = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    explicit Ctx(int device) {
        cudaGetDevice(&prev);
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
        ck(cudaEventCreate(&e0), "cudaEventCreate");
        ck(cudaEventCreate(&e1), "cudaEventCreate");
    }
    ~Ctx() {
        if (s) cudaStreamSynchronize(s);
        if (e0) cudaEventDestroy(e0);
        if (e1) cudaEventDestroy(e1);
        if (s) cudaStreamDestroy(s);
        if (prev >= 0) cudaSetDevice(prev);
    }
    void sync() {
        ck(cudaGetLastError(), "kernel launch");
        ck(cudaStreamSynchronize(s), "device execution");
    }
    void start() { ck(cudaEventRecord(e0, s), "cudaEventRecord"); }
    double stop_ms() {
        ck(cudaEventRecord(e1, s), "cudaEventRecord");
        sync();
        float ms = 0.f;
        ck(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
        return ms;
    }
    template <class T>
    Dev<T> upload(const T* h, size_t count) {
        Dev<T> d(count);
        if (count) ck(cudaMemcpyAsync(d.p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s), "H2D");
        return d;
    }
    template <class T>
    void download(T* h, const T* d, size_t count) {
        if (count) ck(cudaMemcpyAsync(h, d, sizeof(T) * count, cudaMemcpyDeviceToHost, s), "D2H");
        sync();
    }
};

double dev_sumsq(Ctx& cx, const double* v, long long n) {
    const int parts = sumsq_parts(n);
    Dev<double> part(parts), out(1);
    launch_sumsq(v, n, part.p, cx.s);
    launch_reduce_parts(part.p, parts, out.p, cx.s);
    double h = 0.0;
    cx.download(&h, out.p, 1);
    return h;
}

// D = A·B (+ Cin − … when Cin given); A M×K, B K×N, all row-major, packed
void gemm(cudaStream_t s, long long M, long long N, long long K, const double* A, const double* B,
          double* D, const double* Cin = nullptr, double* sq_part = nullptr, bool store = true) {
    GemmArgs g{};
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = K;
    g.B = B;
    g.ldb = N;
    g.b_trans = 0;
    g.D = D;
    g.ldd = N;
    g.Cin = Cin;
    g.ldc = N;
    g.Rold = nullptr;
    g.ldr = 0;
    g.sq_part = sq_part;
    g.diff_part = nullptr;
    g.store = store ? 1 : 0;
    g.sym = 0;
    launch_gemm(g, s);
}

double default_rank_tol(long long rows, long long cols, double sigma_max) {  // decomp.hpp:30-33
    return 8.0 * static_cast<double>(std::max(rows, cols)) * sigma_max * std::ldexp(1.0, -52);
}

// The Jacobi factorisation of one operand, kept on the device.
struct SvdDev {
    long long rows = 0, cols = 0, m_w = 0, n_w = 0;
    bool wide = false;
    Dev<double> Wc;              // n_w × m_w: column j of W = A·V (or Aᵀ·V) as row j
    Dev<double> Vc;              // n_w × n_w: column j of V as row j
    std::vector<double> sigma;   // ‖w_j‖, column order
    std::vector<int> order;      // stable nonincreasing order (decomp.hpp:125-128)
    size_t rank = 0;             // numeric rank at the default cutoff
    int sweeps = 0;

    double sigma_max() const { return sigma.empty() ? 0.0 : sigma[order[0]]; }
    size_t rank_at(double tol) const {  // rank_of (analysis.hpp:54-61)
        if (tol < 0.0) return rank;
        size_t r = 0;
        for (double s : sigma) r += s > tol;
        return r;
    }
};

void svd_device(Ctx& cx, const double* dM, long long rows, long long cols, size_t max_sweeps,
                SvdDev& f) {
    if (rows == 0 || cols == 0) fail(AXB_SHAPE_ERROR, "svd: empty matrix");
    f.rows = rows;
    f.cols = cols;
    f.wide = rows < cols;
    f.m_w = f.wide ? cols : rows;
    f.n_w = f.wide ? rows : cols;
    const long long m = f.m_w, n = f.n_w;
    f.Wc.alloc((size_t)(m * n));
    if (f.wide)  // W = Mᵀ: its columns are M's rows
        ck(cudaMemcpyAsync(f.Wc.p, dM, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, cx.s), "D2D");
    else
        launch_transpose(dM, rows, cols, f.Wc.p, cx.s);
    f.Vc.alloc((size_t)(n * n));
    ck(cudaMemsetAsync(f.Vc.p, 0, sizeof(double) * n * n, cx.s), "memset");
    k_set_diag<<<(unsigned)((n + 255) / 256), 256, 0, cx.s>>>(f.Vc.p, n, 1.0);
    const double null_sq = dev_sumsq(cx, f.Wc.p, m * n) * 1e-30;  // decomp.hpp:74

    const int N = (int)(n + (n & 1));
    Dev<int> flag(1);
    bool converged = false;
    const bool vec = (m & 1) == 0;
    const int grid = jacobi_grid(m, n, N);
    for (size_t sweep = 0; sweep < max_sweeps; ++sweep) {
        ck(cudaMemsetAsync(flag.p, 0, sizeof(int), cx.s), "memset");
        for (int r = 0; r + 1 < N; ++r) {
            if (vec)
                k_jacobi_round<true><<<grid, kJT, 0, cx.s>>>(f.Wc.p, m, f.Vc.p, n, N, r, null_sq, flag.p);
            else
                k_jacobi_round<false><<<grid, kJT, 0, cx.s>>>(f.Wc.p, m, f.Vc.p, n, N, r, null_sq, flag.p);
        }
        int h = 0;
        cx.download(&h, flag.p, 1);
        f.sweeps = (int)sweep + 1;
        if (!h) {
            converged = true;
            break;
        }
    }
    if (!converged) fail(AXB_DECOMPOSITION_ERROR, "svd: Jacobi sweeps exceeded cap");

    Dev<double> sig((size_t)n);
    k_row_norms<<<(unsigned)n, kJT, 0, cx.s>>>(f.Wc.p, m, sig.p);
    f.sigma.resize((size_t)n);
    cx.download(f.sigma.data(), sig.p, (size_t)n);
    f.order.resize((size_t)n);
    std::iota(f.order.begin(), f.order.end(), 0);
    std::stable_sort(f.order.begin(), f.order.end(),
                     [&](int a, int b) { return f.sigma[a] > f.sigma[b]; });
    const double cutoff = default_rank_tol(rows, cols, f.sigma_max());
    f.rank = 0;
    for (size_t j = 0; j < (size_t)n; ++j)
        if (f.sigma[f.order[j]] > cutoff) f.rank = j + 1;
}

// P (cols × rows) = Σ_{σ_k > tol} v_k w_kᵀ / σ_k² (tall) or w_k v_kᵀ / σ_k² (wide);
// tol < 0 selects the default cutoff (decomp.hpp:163).
void pinv_device(Ctx& cx, const SvdDev& f, double tol, double* dP) {
    if (tol < 0.0) tol = default_rank_tol(f.rows, f.cols, f.sigma_max());
    const long long nw = f.n_w;
    std::vector<double> d((size_t)nw);
    for (long long j = 0; j < nw; ++j) {
        const double s = f.sigma[(size_t)j];
        d[(size_t)j] = (s <= tol) ? 0.0 : (1.0 / s) / s;  // decomp.hpp:168-170
    }
    Dev<double> dd = cx.upload(d.data(), d.size());
    const double* X = f.wide ? f.Wc.p : f.Vc.p;  // nw × a, a = cols
    const double* Y = f.wide ? f.Vc.p : f.Wc.p;  // nw × b, b = rows
    const long long a = f.cols, b = f.rows;
    Dev<double> Xt((size_t)(a * nw)), Ys((size_t)(nw * b));
    launch_transpose(X, nw, a, Xt.p, cx.s);
    ck(cudaMemcpyAsync(Ys.p, Y, sizeof(double) * nw * b, cudaMemcpyDeviceToDevice, cx.s), "D2D");
    k_scale_rows<<<grid_for(nw * b), 256, 0, cx.s>>>(Ys.p, nw, b, dd.p);
    gemm(cx.s, a, b, nw, Xt.p, Ys.p, dP);
    cx.sync();
}

// complete rows [from, n) of Uc (n × len, orthonormal rows) with unit vectors
// orthogonal to the rows before them: detail::complete_orthonormal_columns
// (decomp.hpp:39-65) — candidates e_0, e_1, … projected twice, kept when the
// remaining norm exceeds 0.5 (classical Gram–Schmidt per pass on the device)
void complete_rows(Ctx& cx, double* Uc, long long n, long long len, long long from) {
    if (from >= n) return;
    Dev<double> cand((size_t)len), dots((size_t)std::max<long long>(n, 1));
    long long next_basis = 0;
    const double one = 1.0;
    for (long long j = from; j < n; ++j) {
        for (;; ++next_basis) {
            if (next_basis == len) fail(AXB_DECOMPOSITION_ERROR, "svd: failed to complete orthonormal basis");
            ck(cudaMemsetAsync(cand.p, 0, sizeof(double) * len, cx.s), "memset");
            ck(cudaMemcpyAsync(cand.p + next_basis, &one, sizeof(double), cudaMemcpyHostToDevice, cx.s), "H2D");
            for (int pass = 0; pass < 2 && j > 0; ++pass) {
                k_gs_dots<<<(unsigned)j, kJT, 0, cx.s>>>(Uc, len, cand.p, dots.p);
                k_gs_sub<<<(unsigned)((len + 255) / 256), 256, 0, cx.s>>>(Uc, len, (int)j, dots.p, cand.p);
            }
            const double nrm = std::sqrt(dev_sumsq(cx, cand.p, len));
            if (nrm > 0.5) {
                k_div_copy<<<(unsigned)((len + 255) / 256), 256, 0, cx.s>>>(cand.p, len, nrm, Uc + j * len);
                ++next_basis;
                break;
            }
        }
    }
    cx.sync();
}

thread_local uint64_t g_sweeps[2] = {0, 0};
thread_local double g_device_ms = 0.0;

int guarded(const std::function<void()>& f) {
    try {
        f();
        handleless_error().clear();
        return AXB_OK;
    } catch (const Fail& e) {
        handleless_error() = e.msg;
        return e.code;
    } catch (const std::bad_alloc&) {
        handleless_error() = "host allocation failed";
        return AXB_CAPACITY_ERROR;
    } catch (const std::exception& e) {
        handleless_error() = e.what();
        return AXB_CUDA_ERROR;
    }
}

struct Operand {
    std::vector<double> host;  // CSR expansion
    const double* p = nullptr;
    long long rows = 0, cols = 0;
};

Operand operand(const axb_matrix* M, const char* name) {
    if (!M) fail(AXB_CONFIG_ERROR, "%s: null matrix", name);
    Operand o;
    const int st = expand_matrix(M, o.host, name);
    if (st) throw Fail{st, handleless_error()};
    o.p = M->kind == 1 ? o.host.data() : M->dense;
    o.rows = (long long)M->rows;
    o.cols = (long long)M->cols;
    if (!o.p && o.rows * o.cols) fail(AXB_CONFIG_ERROR, "%s: null data", name);
    return o;
}

}  // namespace
}  // namespace axb_dev

using namespace axb_dev;

extern "C" {

int axb_svd(const double* M, uint64_t rows, uint64_t cols, uint64_t max_sweeps, int32_t device,
            double* U, double* sigma, double* V, uint64_t* numeric_rank) {
    return guarded([&] {
        if (rows == 0 || cols == 0) fail(AXB_SHAPE_ERROR, "svd: empty matrix");
        Ctx cx(device);
        Dev<double> dM = cx.upload(M, (size_t)(rows * cols));
        cx.start();
        SvdDev f;
        svd_device(cx, dM.p, (long long)rows, (long long)cols, (size_t)max_sweeps, f);
        const long long m = f.m_w, n = f.n_w;
        std::vector<int> ord(f.order);
        std::vector<double> sv((size_t)n);
        for (long long j = 0; j < n; ++j) sv[(size_t)j] = f.sigma[(size_t)ord[(size_t)j]];
        if (U || V) {
            Dev<int> dord = cx.upload(ord.data(), ord.size());
            Dev<double> dsv = cx.upload(sv.data(), sv.size());
            // F_U (sorted, normalised, completed) and F_V (sorted), as rows
            Dev<double> Fu((size_t)(n * m)), Fv((size_t)(n * n)), T((size_t)std::max(n * m, n * n));
            ck(cudaMemsetAsync(Fu.p, 0, sizeof(double) * n * m, cx.s), "memset");
            if (f.rank)
                k_gather_rows<<<grid_for((long long)f.rank * m), 256, 0, cx.s>>>(
                    f.Wc.p, m, dord.p, dsv.p, (long long)f.rank, Fu.p);
            complete_rows(cx, Fu.p, n, m, (long long)f.rank);
            k_gather_rows<<<grid_for(n * n), 256, 0, cx.s>>>(f.Vc.p, n, dord.p, nullptr, n, Fv.p);
            // tall: U = F_U (rows × n), V = F_V; wide: swapped (decomp.hpp:155)
            double* u_out = f.wide ? V : U;
            double* v_out = f.wide ? U : V;
            if (u_out) {
                launch_transpose(Fu.p, n, m, T.p, cx.s);
                cx.download(u_out, T.p, (size_t)(m * n));
            }
            if (v_out) {
                launch_transpose(Fv.p, n, n, T.p, cx.s);
                cx.download(v_out, T.p, (size_t)(n * n));
            }
        }
        g_device_ms = cx.stop_ms();
        g_sweeps[0] = (uint64_t)f.sweeps;
        g_sweeps[1] = 0;
        if (sigma) std::memcpy(sigma, sv.data(), sizeof(double) * (size_t)n);
        if (numeric_rank) *numeric_rank = f.rank;
    });
}

int axb_pseudoinverse(const double* M, uint64_t rows, uint64_t cols, double rank_tol,
                      int32_t device, double* P) {
    return guarded([&] {
        if (rows == 0 || cols == 0) fail(AXB_SHAPE_ERROR, "svd: empty matrix");
        Ctx cx(device);
        Dev<double> dM = cx.upload(M, (size_t)(rows * cols));
        cx.start();
        SvdDev f;
        svd_device(cx, dM.p, (long long)rows, (long long)cols, 64, f);
        Dev<double> dP((size_t)(rows * cols));
        pinv_device(cx, f, rank_tol, dP.p);
        g_device_ms = cx.stop_ms();
        g_sweeps[0] = (uint64_t)f.sweeps;
        g_sweeps[1] = 0;
        cx.download(P, dP.p, (size_t)(rows * cols));
    });
}

int axb_reference_solution(const axb_matrix* A, const axb_matrix* B, const double* C,
                           double rank_tol, int32_t device, double* X, int32_t* kind,
                           double* residual_check) {
    return guarded([&] {
        Operand a = operand(A, "A"), b = operand(B, "B");
        const long long m = a.rows, p = a.cols, q = b.rows, n = b.cols;
        if (!m || !p || !q || !n) fail(AXB_SHAPE_ERROR, "svd: empty matrix");
        if (!C) fail(AXB_CONFIG_ERROR, "C: null data");
        Ctx cx(device);
        Dev<double> dA = cx.upload(a.p, (size_t)(m * p)), dB = cx.upload(b.p, (size_t)(q * n)),
                    dC = cx.upload(C, (size_t)(m * n));
        cx.start();
        Dev<double> PA((size_t)(p * m)), PB((size_t)(n * q));
        int32_t k;
        {
        SvdDev fa, fb;
        svd_device(cx, dA.p, m, p, 64, fa);
        svd_device(cx, dB.p, q, n, 64, fb);
        g_sweeps[0] = (uint64_t)fa.sweeps;
        g_sweeps[1] = (uint64_t)fb.sweeps;
        const size_t rank_a = fa.rank_at(rank_tol), rank_b = fb.rank_at(rank_tol);
        const bool a_full_col = rank_a == (size_t)p, a_full_row = rank_a == (size_t)m;
        const bool b_full_col = rank_b == (size_t)n, b_full_row = rank_b == (size_t)q;
        double tol;
        if (a_full_col && b_full_row) {
            k = AXB_REF_UNIQUE_FULL_RANK;
            tol = 0.0;  // the LU solves invert every positive σ
        } else if (a_full_row && b_full_col) {
            k = AXB_REF_LEAST_NORM_FULL_ROW_COL;
            tol = 0.0;
        } else {
            k = AXB_REF_LEAST_NORM_GENERAL;
            tol = rank_tol;
        }
        pinv_device(cx, fa, tol, PA.p);
        pinv_device(cx, fb, tol, PB.p);
        }  // the factors are released before the products
        Dev<double> T((size_t)(p * n)), dX((size_t)(p * q));
        gemm(cx.s, p, n, m, PA.p, dC.p, T.p);   // A⁺·C
        gemm(cx.s, p, q, n, T.p, PB.p, dX.p);   // (A⁺·C)·B⁺
        // residual_check = ‖C − (A·X*)·B‖_F (analysis.hpp:86)
        Dev<double> AX((size_t)(m * q));
        gemm(cx.s, m, q, p, dA.p, dX.p, AX.p);
        const int parts = gemm_num_ctas(m, n);
        Dev<double> part((size_t)parts), out(1);
        gemm(cx.s, m, n, q, AX.p, dB.p, nullptr, dC.p, part.p, false);
        launch_reduce_parts(part.p, parts, out.p, cx.s);
        double res_sq = 0.0;
        cx.download(&res_sq, out.p, 1);
        const double c_fro = std::sqrt(dev_sumsq(cx, dC.p, m * n));
        g_device_ms = cx.stop_ms();
        const double res = std::sqrt(res_sq);
        if (kind) *kind = k;
        if (residual_check) *residual_check = res;
        if (res > 1e-8 * (1.0 + c_fro))  // kConsistencyGuardScale (analysis.hpp:16, :88-90)
            fail(AXB_DOMAIN_ERROR, "reference_solution: system is not consistent (residual %f)", res);
        cx.download(X, dX.p, (size_t)(p * q));
    });
}

int axb_bk_limit(const axb_matrix* A, const axb_matrix* B, const double* C, const double* X0,
                 int32_t device, double* X) {
    return guarded([&] {
        Operand a = operand(A, "A"), b = operand(B, "B");
        const long long m = a.rows, p = a.cols, q = b.rows, n = b.cols;
        if (!m || !p || !q || !n) fail(AXB_SHAPE_ERROR, "svd: empty matrix");
        if (!C || !X0) fail(AXB_CONFIG_ERROR, "C/X0: null data");
        Ctx cx(device);
        Dev<double> dA = cx.upload(a.p, (size_t)(m * p)), dB = cx.upload(b.p, (size_t)(q * n)),
                    dC = cx.upload(C, (size_t)(m * n)), dX0 = cx.upload(X0, (size_t)(p * q));
        cx.start();
        Dev<double> PA((size_t)(p * m)), PB((size_t)(n * q));
        {
            SvdDev fa, fb;
            svd_device(cx, dA.p, m, p, 64, fa);
            pinv_device(cx, fa, -1.0, PA.p);
            svd_device(cx, dB.p, q, n, 64, fb);
            pinv_device(cx, fb, -1.0, PB.p);
            g_sweeps[0] = (uint64_t)fa.sweeps;
            g_sweeps[1] = (uint64_t)fb.sweeps;
        }
        // A⁺CB⁺ + X0 − A⁺(A·X0·B)B⁺ = X0 + A⁺·(C − A·X0·B)·B⁺ (analysis.hpp:101-103)
        Dev<double> AX((size_t)(m * q)), D((size_t)(m * n)), T((size_t)(p * n)), F((size_t)(p * q));
        gemm(cx.s, m, q, p, dA.p, dX0.p, AX.p);
        gemm(cx.s, m, n, q, AX.p, dB.p, D.p, dC.p);
        gemm(cx.s, p, n, m, PA.p, D.p, T.p);
        gemm(cx.s, p, q, n, T.p, PB.p, F.p);
        k_add<<<grid_for(p * q), 256, 0, cx.s>>>(dX0.p, F.p, p * q, F.p);
        g_device_ms = cx.stop_ms();
        cx.download(X, F.p, (size_t)(p * q));
    });
}

int axb_rrn(const double* Xk, const double* ref, uint64_t len, int32_t device, double* out) {
    return guarded([&] {
        Ctx cx(device);
        Dev<double> a = cx.upload(Xk, (size_t)len), b = cx.upload(ref, (size_t)len);
        const int parts = grid_for((long long)len);
        Dev<double> part((size_t)(2 * parts));
        k_rrn_parts<<<parts, kJT, 0, cx.s>>>(a.p, b.p, (long long)len, part.p);
        std::vector<double> h((size_t)(2 * parts));
        cx.download(h.data(), part.p, h.size());
        double d = 0.0, r = 0.0;
        for (int i = 0; i < parts; ++i) {
            d += h[(size_t)i];
            r += h[(size_t)(parts + i)];
        }
        if (r == 0.0) fail(AXB_DOMAIN_ERROR, "rrn: zero reference");
        *out = d / r;
    });
}

int axb_analysis_stats(uint64_t sweeps[2], double* device_ms) {
    if (sweeps) {
        sweeps[0] = g_sweeps[0];
        sweeps[1] = g_sweeps[1];
    }
    if (device_ms) *device_ms = g_device_ms;
    return AXB_OK;
}

}  // extern "C"
