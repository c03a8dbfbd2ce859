// axb_solver.cu — host C++ engine behind the C-ABI (include/axb_b200.h).
//
// Mirrors axb::Solver<DenseMatrix,DenseMatrix> (solver.hpp:143-515): the same
// constructor checks and initialisation order (:146-192), the same run() loop
// with its confirm/resync and refresh-checkpoint schedule (:337-372), the same
// public selection and metric methods.  The iteration itself runs on the
// device (axb_iter.cu), batched into CUDA graphs; the host only intervenes at
// batch boundaries, refresh checkpoints and stop confirmations.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <condition_variable>
#include <mutex>
#include <set>
#include <thread>

#include "../../include/axb_b200.h"
#include "axb_device.cuh"
#include "axb_nccl.cuh"

namespace axb_nccl {
const Api* api(const char** why) {
    static Api a;
    static int state = 0;  // 0 untried, 1 ok, −1 failed
    static const char* reason = "";
    if (state == 0) {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            state = -1;
            reason = "libnccl.so.2 not found";
        } else {
            a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
            a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
            a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
            a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
            a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
            a.GetErrorString =
                reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
            a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(dlsym(h, "ncclGroupStart"));
            a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(dlsym(h, "ncclGroupEnd"));
            const bool ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllReduce &&
                            a.AllGather && a.GetErrorString && a.GroupStart && a.GroupEnd;
            state = ok ? 1 : -1;
            if (!ok) reason = "libnccl.so.2 lacks a required symbol";
        }
    }
    if (why) *why = reason;
    return state == 1 ? &a : nullptr;
}

// ---- in-process emulation of the collectives (test infrastructure) ----------
// `world` ranks as host threads of ONE process on ONE GPU, each with its own
// solver handle and stream.  A collective synchronises the caller's stream,
// meets the other ranks at a host barrier, lets rank 0 combine the buffers (sums
// in rank order, gathers by copy), and meets them again — so no rank's kernel
// ever waits on another rank's kernel, and the sharded code path (every kernel,
// every offset and owner decision) runs with world > 1 where only one GPU is
// available.  Solvers on an emulated communicator launch iterations directly
// (a host-synchronising collective cannot be captured into a CUDA graph).
struct EmuGroup {
    int world = 1;
    int alive = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t gen = 0;
    struct Slot {
        const void* send;
        void* recv;
        size_t count;
    };
    std::vector<Slot> slots;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const uint64_t g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
struct EmuComm {
    EmuGroup* grp;
    int rank;
};
std::mutex g_emu_mu;
std::set<const void*> g_emu_comms;

bool is_emulated(const void* comm) {
    std::lock_guard<std::mutex> lk(g_emu_mu);
    return g_emu_comms.count(comm) != 0;
}

ncclResult_t emu_allreduce(const void* send, void* recv, size_t count, ncclDataType_t dt,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
    if (dt != ncclFloat64 || op != ncclSum) return ncclInvalidArgument;
    auto* c = reinterpret_cast<EmuComm*>(comm);
    EmuGroup* G = c->grp;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ncclUnhandledCudaError;
    G->slots[c->rank] = {send, recv, count};
    G->barrier();
    ncclResult_t rc = ncclSuccess;
    if (c->rank == 0) {
        std::vector<double> acc(count, 0.0), tmp(count);
        for (int r = 0; r < G->world && rc == ncclSuccess; ++r) {
            if (cudaMemcpy(tmp.data(), G->slots[r].send, count * sizeof(double),
                           cudaMemcpyDeviceToHost) != cudaSuccess)
                rc = ncclUnhandledCudaError;
            for (size_t i = 0; i < count; ++i) acc[i] += tmp[i];
        }
        for (int r = 0; r < G->world && rc == ncclSuccess; ++r)
            if (cudaMemcpy(G->slots[r].recv, acc.data(), count * sizeof(double),
                           cudaMemcpyHostToDevice) != cudaSuccess)
                rc = ncclUnhandledCudaError;
        if (cudaDeviceSynchronize() != cudaSuccess) rc = ncclUnhandledCudaError;
    }
    G->barrier();
    return rc;
}

ncclResult_t emu_allgather(const void* send, void* recv, size_t count, ncclDataType_t dt,
                           ncclComm_t comm, cudaStream_t s) {
    if (dt != ncclFloat64) return ncclInvalidArgument;
    auto* c = reinterpret_cast<EmuComm*>(comm);
    EmuGroup* G = c->grp;
    if (cudaStreamSynchronize(s) != cudaSuccess) return ncclUnhandledCudaError;
    G->slots[c->rank] = {send, recv, count};
    G->barrier();
    ncclResult_t rc = ncclSuccess;
    if (c->rank == 0) {
        const size_t bytes = count * sizeof(double);
        for (int r = 0; r < G->world; ++r)
            for (int t = 0; t < G->world; ++t) {
                char* dst = static_cast<char*>(G->slots[t].recv) + (size_t)r * bytes;
                if (dst == G->slots[r].send) continue;  // in place
                if (cudaMemcpy(dst, G->slots[r].send, bytes, cudaMemcpyDeviceToDevice) !=
                    cudaSuccess)
                    rc = ncclUnhandledCudaError;
            }
        if (cudaDeviceSynchronize() != cudaSuccess) rc = ncclUnhandledCudaError;
    }
    G->barrier();
    return rc;
}

ncclResult_t emu_destroy(ncclComm_t comm) {
    auto* c = reinterpret_cast<EmuComm*>(comm);
    std::lock_guard<std::mutex> lk(g_emu_mu);
    g_emu_comms.erase(c);
    EmuGroup* G = c->grp;
    delete c;
    if (--G->alive == 0) delete G;
    return ncclSuccess;
}

// the emulated collectives complete synchronously, one after another: a group
// needs no fusing
ncclResult_t emu_group() { return ncclSuccess; }

const char* emu_error(ncclResult_t r) {
    return r == ncclSuccess ? "ok" : "emulated collective failed";
}

const Api* emulated_api() {
    static Api e;
    static bool init = false;
    std::lock_guard<std::mutex> lk(g_emu_mu);
    if (!init) {
        e.AllReduce = emu_allreduce;
        e.AllGather = emu_allgather;
        e.CommDestroy = emu_destroy;
        e.GetErrorString = emu_error;
        e.GroupStart = emu_group;
        e.GroupEnd = emu_group;
        init = true;
    }
    return &e;
}

void emulated_group(int world, void** comms) {
    auto* G = new EmuGroup;
    G->world = world;
    G->alive = world;
    G->slots.resize(world);
    std::lock_guard<std::mutex> lk(g_emu_mu);
    for (int r = 0; r < world; ++r) {
        auto* c = new EmuComm{G, r};
        g_emu_comms.insert(c);
        comms[r] = c;
    }
}
}  // namespace axb_nccl

using namespace axb_dev;

namespace {
thread_local std::string g_create_err;  // message of the last handle-less failure

struct AxbError {
    int code;
    std::string msg;
    uint64_t k = 0;
    double val = 0.0;
};

[[noreturn]] void fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    throw AxbError{code, buf};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        if (e == cudaErrorMemoryAllocation)
            fail(AXB_CAPACITY_ERROR, "%s: out of device memory (%s)", what, cudaGetErrorString(e));
        fail(AXB_CUDA_ERROR, "%s: %s", what, cudaGetErrorString(e));
    }
}

// ---- host restatement of decomp.hpp:207-239 (bitwise α for small B) ----
uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

std::vector<double> power_start(size_t dim) {
    std::vector<double> v(dim);
    uint64_t h = 0x6b8f9a37c1d2e4f5ULL;
    for (size_t i = 0; i < dim; ++i) {
        h = splitmix64(h);
        v[i] = 1.0 + 1e-3 * (static_cast<double>(h >> 11) * 0x1.0p-53 - 0.5);
    }
    double nrm = 0.0;
    for (size_t i = 0; i < dim; ++i) nrm = nrm + v[i] * v[i];
    nrm = std::sqrt(nrm);
    for (double& x : v) x /= nrm;
    return v;
}

double spectral_norm_host(const std::vector<double>& b, size_t rows, size_t cols, double tol,
                          size_t max_iter) {
    double fro = 0.0;
    for (double v : b) fro += v * v;
    if (fro == 0.0) fail(AXB_DOMAIN_ERROR, "spectral_norm: zero matrix");
    const bool use_mtm = cols <= rows;
    const size_t dim = use_mtm ? cols : rows, other = use_mtm ? rows : cols;
    std::vector<double> v = power_start(dim), w(dim), t(other);
    auto matvec = [&](const double* x, double* y) {  // matrix.hpp:400-410
        for (size_t i = 0; i < rows; ++i) {
            const double* ri = b.data() + i * cols;
            double s = 0.0;
            for (size_t j = 0; j < cols; ++j) s += ri[j] * x[j];
            y[i] = s;
        }
    };
    auto matvec_t = [&](const double* x, double* y) {  // matrix.hpp:420-430
        for (size_t j = 0; j < cols; ++j) y[j] = 0.0;
        for (size_t i = 0; i < rows; ++i) {
            const double xv = x[i];
            if (xv == 0.0) continue;
            const double* ri = b.data() + i * cols;
            for (size_t j = 0; j < cols; ++j) y[j] += xv * ri[j];
        }
    };
    double lambda = 0.0;
    for (size_t it = 0; it < max_iter; ++it) {
        if (use_mtm) {
            matvec(v.data(), t.data());
            matvec_t(t.data(), w.data());
        } else {
            matvec_t(v.data(), t.data());
            matvec(t.data(), w.data());
        }
        double rayleigh = 0.0, wn = 0.0;
        for (size_t i = 0; i < dim; ++i) rayleigh = rayleigh + v[i] * w[i];
        for (size_t i = 0; i < dim; ++i) wn = wn + w[i] * w[i];
        wn = std::sqrt(wn);
        if (wn == 0.0) return 0.0;
        for (size_t i = 0; i < dim; ++i) v[i] = w[i] / wn;
        if (it > 0 && std::abs(rayleigh - lambda) <= 0.5 * tol * std::abs(rayleigh))
            return std::sqrt(rayleigh);
        lambda = rayleigh;
    }
    AxbError e{AXB_CONVERGENCE_ERROR, "spectral_norm: power iteration did not converge"};
    e.val = std::sqrt(std::abs(lambda));
    throw e;
}

bool trace_point_due(uint64_t k) { return k < 10000 || k % 10 == 0; }  // solver.hpp:136

int env_int(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

// AXB_R_KERNEL=simple selects the register-streaming K2 (A/B comparisons)
bool opt_r_tma() {
    const char* e = std::getenv("AXB_R_KERNEL");
    return !(e && std::strcmp(e, "simple") == 0);
}

// Device → host copy-out for the accessors (get_X / get_R / …).  A plain
// cudaMemcpy into a freshly allocated pageable buffer (numpy.empty) measured
// ~4 GB/s on the box — the driver faults the destination pages in serially — so
// X at config 5 (0.54 GB) took 131 ms.  Large pageable copies therefore run
// through two pinned 32 MB staging chunks: the DMA of chunk c+1 overlaps a
// multi-threaded memcpy of chunk c into the destination.  Pinned or registered
// destinations, and small copies, go straight through cudaMemcpy.
void d2h_copy(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    cudaPointerAttributes pa{};
    const bool pinned =
        cudaPointerGetAttributes(&pa, dst) == cudaSuccess && pa.type == cudaMemoryTypeHost;
    cudaGetLastError();  // an unregistered pointer may leave a sticky-free error code
    constexpr size_t kChunk = size_t(32) << 20;
    if (pinned || bytes < 2 * kChunk) {
        ck(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s), "copy out");
        ck(cudaStreamSynchronize(s), "copy out");
        return;
    }
    static std::mutex mu;
    static char* stage[2] = {nullptr, nullptr};
    std::lock_guard<std::mutex> lock(mu);
    for (auto& b : stage)
        if (!b) ck(cudaMallocHost(reinterpret_cast<void**>(&b), kChunk), "pinned staging");
    cudaEvent_t ev[2];
    for (auto& e : ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            cudaEventDestroy(e[0]);
            cudaEventDestroy(e[1]);
        }
    } eg{ev};
    const size_t nch = (bytes + kChunk - 1) / kChunk;
    auto enqueue = [&](size_t c) {
        const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        ck(cudaMemcpyAsync(stage[c & 1], static_cast<const char*>(src) + off, len,
                           cudaMemcpyDeviceToHost, s), "copy out");
        ck(cudaEventRecord(ev[c & 1], s), "event");
    };
    const unsigned nthr = std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    enqueue(0);
    for (size_t c = 0; c < nch; ++c) {
        if (c + 1 < nch) enqueue(c + 1);  // its staging chunk was drained at step c-1
        ck(cudaEventSynchronize(ev[c & 1]), "copy out");
        const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
        const size_t per = (len / nthr + 63) & ~size_t(63);
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nthr; ++t) {
            const size_t a = std::min(len, t * per), b = std::min(len, a + per);
            if (a < b)
                th.emplace_back([=] {
                    std::memcpy(static_cast<char*>(dst) + off + a, stage[c & 1] + a, b - a);
                });
        }
        for (auto& t : th) t.join();
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count, const char* what) {
        n = count;
        ck(cudaMalloc(&p, sizeof(T) * std::max<size_t>(count, 1)), what);
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// ---- host CSR helpers ----
struct Csr {
    uint64_t rows = 0, cols = 0;
    std::vector<long long> rp;
    std::vector<int> ci;
    std::vector<double> v;
};

Csr csr_of(const axb_matrix* M) {  // validated by create_ex (SparseMatrix::validate)
    Csr c;
    c.rows = M->rows;
    c.cols = M->cols;
    c.rp.assign(M->row_ptr, M->row_ptr + M->rows + 1);
    c.ci.resize(M->nnz);
    for (uint64_t e = 0; e < M->nnz; ++e) c.ci[e] = (int)M->col_idx[e];
    c.v.assign(M->values, M->values + M->nnz);
    return c;
}

// transpose (matrix.hpp's CSR transpose): column-major counting sort, so each
// row of the result lists its entries in ascending original-row order
Csr csr_transpose(const Csr& a) {
    Csr t;
    t.rows = a.cols;
    t.cols = a.rows;
    t.rp.assign(a.cols + 1, 0);
    for (int c : a.ci) ++t.rp[(size_t)c + 1];
    for (uint64_t j = 0; j < a.cols; ++j) t.rp[j + 1] += t.rp[j];
    t.ci.resize(a.ci.size());
    t.v.resize(a.v.size());
    std::vector<long long> pos(t.rp.begin(), t.rp.end() - 1);
    for (uint64_t i = 0; i < a.rows; ++i)
        for (long long e = a.rp[i]; e < a.rp[i + 1]; ++e) {
            const long long d = pos[(size_t)a.ci[e]]++;
            t.ci[d] = (int)i;
            t.v[d] = a.v[e];
        }
    return t;
}

// gram_mmt(const SparseMatrix&) (matrix.hpp:496-535): Gustavson accumulation of
// M·Mᵀ through Mᵀ's rows in the reference's order (acc[j] += m_ik·m_jk over k in
// row i's stored order), exact-zero sums dropped — so G is the reference's G bit
// for bit (host code, no FMA contraction)
Csr gram_csr(const Csr& a) {
    const Csr t = csr_transpose(a);
    Csr g;
    g.rows = g.cols = a.rows;
    g.rp.assign(a.rows + 1, 0);
    std::vector<double> acc(a.rows, 0.0);
    std::vector<char> seen(a.rows, 0);
    std::vector<int> touched;
    for (uint64_t i = 0; i < a.rows; ++i) {
        for (long long e = a.rp[i]; e < a.rp[i + 1]; ++e) {
            const double v = a.v[e];
            const int k = a.ci[e];
            for (long long f = t.rp[k]; f < t.rp[k + 1]; ++f) {
                const int j = t.ci[f];
                if (!seen[j]) {
                    seen[j] = 1;
                    touched.push_back(j);
                }
                acc[j] += v * t.v[f];
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int j : touched) {
            if (acc[j] != 0.0) {
                g.ci.push_back(j);
                g.v.push_back(acc[j]);
            }
            acc[j] = 0.0;
            seen[j] = 0;
        }
        touched.clear();
        g.rp[i + 1] = (long long)g.ci.size();
    }
    return g;
}

template <class T>
void upload(DevBuf<T>& d, const std::vector<T>& h, const char* what, cudaStream_t s) {
    d.alloc(h.size(), what);
    if (!h.empty()) ck(cudaMemcpyAsync(d.p, h.data(), sizeof(T) * h.size(), cudaMemcpyHostToDevice, s), what);
    ck(cudaStreamSynchronize(s), what);  // h is a pageable temporary
}

}  // namespace

struct axb_solver {
    uint64_t m = 0, p = 0, q = 0, n = 0;
    axb_config cfg{};
    axb_options opt{};
    cudaStream_t stream = nullptr;
    DevBuf<double> A, B, C, R, X, Xref, a_sq, rbk_cum, r_sq, G, g, y, z, zpart, xpart, T,
        gemm_sq, gemm_diff, scal, tr_metric, tr_rel, sq_part, gsum, BtB;
    DevBuf<unsigned int> zcnt;
    DevBuf<RowRecord> rrec;
    // CSR operands: A and its Gram G = A·Aᵀ kept sparse (A is never
    // expanded), B as CSR plus Bᵀ for the per-iteration passes (its dense copy
    // serves ‖B‖₂ and the residual GEMM only)
    const axb_matrix* in_A = nullptr;
    const axb_matrix* in_B = nullptr;
    bool sp_a = false, sp_b = false;
    DevBuf<long long> a_rp, g_rp, b_rp, bt_rp, btb_rp;
    DevBuf<int> a_ci, g_ci, b_ci, bt_ci, btb_ci;
    DevBuf<double> a_v, g_v, b_v, bt_v, btb_v;
    uint64_t nnz_a = 0, nnz_g = 0, nnz_b = 0;
    DevBuf<long long> tr_row, forced;
    // row sharding (§8(e))
    bool sharded = false;
    bool emulated = false;  // in-process collective emulation: no graph capture
    int world = 1, rank = 0;
    uint64_t m_g = 0, row0 = 0, p_loc = 0, n_loc = 0;
    ncclComm_t comm = nullptr;
    const axb_nccl::Api* nc = nullptr;
    DevBuf<double> pack, pack_send, recs, a_sq_g, scal_ag;
    DevBuf<int> flags;
    DevBuf<DevState> st;
    DevState* hs = nullptr;  // pinned host mirror
    std::vector<double> a_sq_h;
    double a_fro_sq = 0.0, b_spec = 0.0, alpha = 0.0, c_fro = 0.0, ref_sq = 0.0;
    bool alpha_outside = false, gram_cached = false;
    bool chain_xb = false;  // residual product as A·(X·B) instead of (A·X)·B
    uint64_t k = 0;
    bool sel_valid = false;
    Params P{};
    cudaGraphExec_t graph = nullptr;
    int graph_iters = 32;
    uint64_t trace_cap = 4096;
    long long* h_trace_row = nullptr;
    double* h_trace_metric = nullptr;
    double* h_trace_rel = nullptr;
    std::string err;
    uint64_t err_k = 0;
    double err_val = 0.0;
    // timing
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    bool profiling = false;
    std::vector<cudaEvent_t> prof_ev;
    double loop_ms = 0.0, k2_ms = 0.0, yg_ms = 0.0, zx_ms = 0.0, sel_ms = 0.0;
    double coll_ms[4] = {0.0, 0.0, 0.0, 0.0};  // y allreduce, z allgather, norms allgather, row allreduce
    static constexpr int kProfEv = 9;
    uint64_t k2_launches = 0, kernel_launches = 0;
    uint64_t last_nb = 0;  // iterations armed by the last batch_launch

    ~axb_solver() {
        if (graph) cudaGraphExecDestroy(graph);
        if (hs) cudaFreeHost(hs);
        if (h_trace_row) cudaFreeHost(h_trace_row);
        if (h_trace_metric) cudaFreeHost(h_trace_metric);
        if (h_trace_rel) cudaFreeHost(h_trace_rel);
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        for (auto e : prof_ev) cudaEventDestroy(e);
        if (stream) cudaStreamDestroy(stream);
    }

    // ---------------------------------------------------------------- utils
    void sync(const char* what) {
        ck(cudaGetLastError(), what);
        ck(cudaStreamSynchronize(stream), what);
    }

    void pull_state() {
        ck(cudaGetLastError(), "kernel launch");
        ck(cudaMemcpyAsync(hs, st.p, sizeof(DevState), cudaMemcpyDeviceToHost, stream), "state");
        sync("state sync");
        if (const unsigned long long v = checked_violation())  // -DAXB_CHECKED builds only
            fail(AXB_CUDA_ERROR, "device bounds check failed at axb_iter.cu:%llu", v);
    }

    [[noreturn]] void raise_state() {
        const int code = hs->err_code ? hs->err_code : AXB_CUDA_ERROR;
        AxbError e{code, ""};
        char buf[256];
        switch (code) {
            case AXB_DIVERGENCE_ERROR:
                snprintf(buf, sizeof buf, "divergence at iteration %llu, residual frobenius norm %f",
                         (unsigned long long)hs->err_k, hs->err_val);
                e.k = hs->err_k;
                e.val = hs->err_val;
                break;
            case AXB_DOMAIN_ERROR:
                if (cfg.method == AXB_GRBK || cfg.method == AXB_RGRBK)
                    snprintf(buf, sizeof buf,
                             !(hs->r_fro_sq > 0.0)
                                 ? "greedy threshold: zero residual"
                                 : "greedy selection: residual mass sits on zero rows of A only; "
                                   "the system is inconsistent");
                else if (cfg.method == AXB_BK)
                    snprintf(buf, sizeof buf, "select_cyclic: no nonzero row");
                else
                    snprintf(buf, sizeof buf, "categorical: no positive weight");
                break;
            default: snprintf(buf, sizeof buf, "device error %d", code);
        }
        e.msg = buf;
        // leave the device state runnable for a caller that catches and continues
        launch_ctrl(st.p, k, k, FIN_ITERATION, 0, 1, stream);
        sync("reset");
        throw e;
    }

    double reduce_sumsq(const double* v, uint64_t len) {
        launch_sumsq(v, (long long)len, sq_part.p, stream);
        launch_reduce_parts(sq_part.p, sumsq_parts((long long)len), scal.p, stream);
        double out = 0.0;
        ck(cudaMemcpyAsync(&out, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream), "sumsq");
        sync("sumsq");
        return out;
    }

    // ---------------------------------------------------------------- collectives
    void nccl_ck(ncclResult_t r, const char* what) {
        if (r != ncclSuccess) fail(AXB_CUDA_ERROR, "%s: %s", what, nc->GetErrorString(r));
    }
    void allgather_inplace(double* buf, size_t count) {  // buf holds world × count
        nccl_ck(nc->AllGather(buf + (size_t)rank * count, buf, count, ncclFloat64, comm, stream),
                "ncclAllGather");
    }
    void allreduce(const double* send, double* recv, size_t count) {
        nccl_ck(nc->AllReduce(send, recv, count, ncclFloat64, ncclSum, comm, stream),
                "ncclAllReduce");
    }
    // every shard's ‖R_l‖² slice into the global r_sq and every shard's record
    // {Σ‖R_l‖², max ratio, argmax, ‖X−X_ref‖² part} into recs: one NCCL group, so
    // one fused collective launch
    void gather_norms() {
        nccl_ck(nc->GroupStart(), "ncclGroupStart");
        allgather_inplace(r_sq.p, m);
        allgather_inplace(recs.p, 4);
        nccl_ck(nc->GroupEnd(), "ncclGroupEnd");
    }
    // Σ over ranks in rank order of a host scalar (identical on every rank)
    double global_sum(double local) {
        if (!sharded) return local;
        ck(cudaMemcpyAsync(scal_ag.p + rank, &local, sizeof(double), cudaMemcpyHostToDevice, stream),
           "global sum");
        allgather_inplace(scal_ag.p, 1);
        std::vector<double> v(world);
        ck(cudaMemcpyAsync(v.data(), scal_ag.p, sizeof(double) * world, cudaMemcpyDeviceToHost,
                           stream), "global sum");
        sync("global sum");
        double acc = 0.0;
        for (double x : v) acc += x;
        return acc;
    }
    // all ranks' rows of X into every rank's full X (p_loc rows per rank)
    void gather_X() {
        if (sharded) allgather_inplace(X.p, (size_t)p_loc * q);
    }

    // ---------------------------------------------------------------- init
    void create(const double* A_in, const double* B_in, const double* C_in, const double* X0_in) {
        // Method::validate (solver.hpp:30-38)
        if (cfg.method < AXB_BK || cfg.method > AXB_MWRBK) fail(AXB_CONFIG_ERROR, "unknown method");
        if (cfg.method == AXB_RGRBK) {
            if (!cfg.has_theta) fail(AXB_CONFIG_ERROR, "rgrbk requires theta");
            if (!(cfg.theta > 0.0 && cfg.theta < 1.0))
                fail(AXB_CONFIG_ERROR, "theta must lie strictly in (0, 1)");
        } else if (cfg.has_theta) {
            fail(AXB_CONFIG_ERROR, "theta is only valid for rgrbk");
        }
        if (cfg.alpha_rule < AXB_ALPHA_SAFE || cfg.alpha_rule > AXB_ALPHA_FIXED)
            fail(AXB_CONFIG_ERROR, "unknown alpha rule");
        if (m == 0 || p == 0) fail(AXB_SHAPE_ERROR, "row_sq_norms: empty matrix");
        if (q == 0 || n == 0) fail(AXB_SHAPE_ERROR, "spectral_norm: empty matrix");
        if (opt.nccl_comm) {
            sharded = true;
            world = std::max(1, opt.world_size);
            rank = opt.rank;
            m_g = opt.m_global ? opt.m_global : m * (uint64_t)world;
            row0 = opt.row_offset;
            const char* why = "";
            emulated = axb_nccl::is_emulated(opt.nccl_comm);
            nc = emulated ? axb_nccl::emulated_api() : axb_nccl::api(&why);
            if (!nc) fail(AXB_CUDA_ERROR, "row sharding needs NCCL: %s", why);
            comm = static_cast<ncclComm_t>(opt.nccl_comm);
            if (rank < 0 || rank >= world) fail(AXB_CONFIG_ERROR, "rank %d outside [0, %d)", rank, world);
            if (m_g != m * (uint64_t)world || row0 != m * (uint64_t)rank)
                fail(AXB_CONFIG_ERROR,
                     "row sharding needs equal contiguous shards: m_global = world·m and "
                     "row_offset = rank·m");
        } else if (opt.world_size > 1) {
            fail(AXB_CONFIG_ERROR, "world_size > 1 needs an NCCL communicator (opt.nccl_comm)");
        } else {
            m_g = m;
            row0 = 0;
        }
        p_loc = (p + world - 1) / world;
        n_loc = (n + world - 1) / world;
        if (n_loc & 1) ++n_loc;
        if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN && !cfg.reference)
            fail(AXB_CONFIG_ERROR, "solution_rrn stopping needs a reference solution");

        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            fail(AXB_CUDA_ERROR, "no CUDA device visible (this build has no CPU fallback)");
        ck(cudaSetDevice(opt.device), "cudaSetDevice");
        cudaDeviceProp prop{};
        ck(cudaGetDeviceProperties(&prop, opt.device), "cudaGetDeviceProperties");
        if (prop.major < 10)
            fail(AXB_CUDA_ERROR, "device %d is sm_%d%d; the kernels are built for sm_100a",
                 opt.device, prop.major, prop.minor);
        ck(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking), "stream");
        ck(cudaEventCreate(&ev0), "event");
        ck(cudaEventCreate(&ev1), "event");
        ck(cudaMallocHost(&hs, sizeof(DevState)), "pinned state");
        if (opt.graph_iters > 0) graph_iters = opt.graph_iters;
        ck(cudaMallocHost(&h_trace_row, sizeof(long long) * trace_cap), "pinned trace");
        ck(cudaMallocHost(&h_trace_metric, sizeof(double) * trace_cap), "pinned trace");
        ck(cudaMallocHost(&h_trace_rel, sizeof(double) * trace_cap), "pinned trace");

        const cudaMemcpyKind kind =
            opt.inputs_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
        // device inputs may still be being written by the caller's work on any of
        // its streams (e.g. C = A·X*·B just queued on torch's current stream); the
        // copy stream below is non-blocking and would not wait for it, so order
        // the copies after everything already queued on this device
        if (opt.inputs_on_device) ck(cudaDeviceSynchronize(), "order after the caller's work");
        // inputs arrive on a copy stream in the order they are needed; the
        // compute stream waits per input, so ‖B‖₂ (and G) overlap the C copy.
        // Each buffer is allocated just before its copy is queued, so mapping the
        // later ones (C, X, R: 35 GB at config 5) overlaps the earlier copies
        sp_a = in_A && in_A->kind == 1;
        sp_b = in_B && in_B->kind == 1;
        if (sp_a || sp_b) {
            if (sharded) fail(AXB_CONFIG_ERROR, "row sharding takes dense operands");
            if (opt.inputs_on_device) fail(AXB_CONFIG_ERROR, "CSR operands are host arrays");
            if ((sp_a && (in_A->cols > 0x7fffffffull || in_A->rows > 0x7fffffffull)) ||
                (sp_b && (in_B->cols > 0x7fffffffull || in_B->rows > 0x7fffffffull)))
                fail(AXB_CAPACITY_ERROR, "CSR dimensions above 2^31");
        }
        if (!sp_a) A.alloc(m * p, "A");
        cudaStream_t cs = nullptr;
        ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "copy stream");
        cudaEvent_t evA, evB, evRest;
        ck(cudaEventCreateWithFlags(&evA, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&evB, cudaEventDisableTiming), "event");
        ck(cudaEventCreateWithFlags(&evRest, cudaEventDisableTiming), "event");
        struct Guard {
            cudaStream_t s;
            cudaEvent_t a, b, c;
            ~Guard() {
                cudaStreamSynchronize(s);
                cudaEventDestroy(a);
                cudaEventDestroy(b);
                cudaEventDestroy(c);
                cudaStreamDestroy(s);
            }
        } guard{cs, evA, evB, evRest};
        if (!sp_a) ck(cudaMemcpyAsync(A.p, A_in, sizeof(double) * m * p, kind, cs), "copy A");
        ck(cudaEventRecord(evA, cs), "event");
        B.alloc(q * n, "B");
        ck(cudaMemcpyAsync(B.p, B_in, sizeof(double) * q * n, kind, cs), "copy B");
        ck(cudaEventRecord(evB, cs), "event");
        C.alloc(m * n, "C");
        ck(cudaMemcpyAsync(C.p, C_in, sizeof(double) * m * n, kind, cs), "copy C");
        X.alloc(p_loc * world * q, "X");
        if (p_loc * world > p)  // X pad, before the X0 copy on the same stream
            ck(cudaMemsetAsync(X.p, 0, sizeof(double) * p_loc * world * q, cs), "X pad");
        if (X0_in)
            ck(cudaMemcpyAsync(X.p, X0_in, sizeof(double) * p * q, kind, cs), "copy X0");
        else
            ck(cudaMemsetAsync(X.p, 0, sizeof(double) * p * q, cs), "zero X0");
        if (cfg.reference) {
            Xref.alloc(p * q, "Xref");
            ck(cudaMemcpyAsync(Xref.p, cfg.reference, sizeof(double) * p * q, kind, cs),
               "copy reference");
        }
        ck(cudaEventRecord(evRest, cs), "event");
        R.alloc(m * n, "R");
        ck(cudaStreamWaitEvent(stream, evA, 0), "wait A");
        a_sq.alloc(m, "a_sq");
        rbk_cum.alloc(m_g, "rbk_cum");
        // sharded: the global ‖R_l‖² (allgathered each iteration); this rank's
        // kernels write their rows in place at row0
        r_sq.alloc(sharded ? m_g : m, "r_sq");
        scal.alloc(4, "scalars");
        if (sharded) {
            a_sq_g.alloc(m_g, "a_sq global");
            scal_ag.alloc(world, "scalar allgather");
            pack.alloc(n + p + 2, "pack");
            pack_send.alloc(n + p + 2, "pack send");
            ck(cudaMemsetAsync(pack_send.p, 0, sizeof(double) * (n + p + 2), stream), "pack");
            recs.alloc(4 * (size_t)world, "records");
        }
        sq_part.alloc(sumsq_parts((long long)std::max({m * n, q * n, p * q, m * p})), "parts");

        // a_sq_ = row_sq_norms(A); a_fro_sq_; rbk_cumsum_ (solver.hpp:156-166), sequential
        if (sp_a) {
            // CSR A: RowView::sq_norm over the stored entries, in order (host), and
            // the CSR arrays the iteration and the residual products read
            const Csr ah = csr_of(in_A);
            nnz_a = ah.v.size();
            std::vector<double> as(m, 0.0);
            for (uint64_t i = 0; i < m; ++i) {
                double sacc = 0.0;
                for (long long e = ah.rp[i]; e < ah.rp[i + 1]; ++e) sacc += ah.v[e] * ah.v[e];
                as[i] = sacc;
            }
            ck(cudaMemcpyAsync(a_sq.p, as.data(), sizeof(double) * m, cudaMemcpyHostToDevice, stream),
               "a_sq");
            upload(a_rp, ah.rp, "A row_ptr", stream);
            upload(a_ci, ah.ci, "A col_idx", stream);
            upload(a_v, ah.v, "A values", stream);
            const Csr gh = gram_csr(ah);  // gram_ = gram_mmt(A) (solver.hpp:171)
            nnz_g = gh.v.size();
            upload(g_rp, gh.rp, "G row_ptr", stream);
            upload(g_ci, gh.ci, "G col_idx", stream);
            upload(g_v, gh.v, "G values", stream);
        } else {
            launch_row_sq_seq(A.p, (long long)m, (long long)p, a_sq.p, stream);
        }
        if (sp_b) {
            const Csr bh = csr_of(in_B);
            nnz_b = bh.v.size();
            const Csr bt = csr_transpose(bh);
            upload(b_rp, bh.rp, "B row_ptr", stream);
            upload(b_ci, bh.ci, "B col_idx", stream);
            upload(b_v, bh.v, "B values", stream);
            upload(bt_rp, bt.rp, "B^T row_ptr", stream);
            upload(bt_ci, bt.ci, "B^T col_idx", stream);
            upload(bt_v, bt.v, "B^T values", stream);
            // btb_ = BᵀB (solver.hpp:172) as the Gram of Bᵀ: entry (c, c') sums
            // B_jc·B_jc' over ascending j, the reference's matmul order
            const Csr btb = gram_csr(bt);
            upload(btb_rp, btb.rp, "B^T B row_ptr", stream);
            upload(btb_ci, btb.ci, "B^T B col_idx", stream);
            upload(btb_v, btb.v, "B^T B values", stream);
        }
        const double* a_all = a_sq.p;
        if (sharded) {  // every rank holds all ‖A_i‖² (BK/RBK selection, ‖A‖²_F, CDF)
            ck(cudaMemcpyAsync(a_sq_g.p + row0, a_sq.p, sizeof(double) * m,
                               cudaMemcpyDeviceToDevice, stream), "a_sq slot");
            allgather_inplace(a_sq_g.p, m);
            a_all = a_sq_g.p;
        }
        launch_cumsum_seq(a_all, (long long)m_g, rbk_cum.p, scal.p, stream);
        a_sq_h.resize(m);
        ck(cudaMemcpyAsync(a_sq_h.data(), a_sq.p, sizeof(double) * m, cudaMemcpyDeviceToHost,
                           stream), "a_sq");
        ck(cudaMemcpyAsync(&a_fro_sq, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream),
           "a_fro");
        sync("init norms");
        if (a_fro_sq == 0.0) fail(AXB_DOMAIN_ERROR, "solve: A is the zero matrix");

        // b_spec_ = spectral_norm(B); resolve_alpha() (solver.hpp:168-169, :439-456)
        ck(cudaStreamWaitEvent(stream, evB, 0), "wait B");
        if (opt.alpha_override > 0.0) {
            alpha = opt.alpha_override;
            b_spec = 0.0;
        } else {
            const size_t cap = opt.spectral_max_iter ? opt.spectral_max_iter : 5000;
            bool on_dev = opt.spectral_on_device == 1 ||
                          (opt.spectral_on_device < 0 && q * n > (1ull << 20));
            if (on_dev) {
                b_spec = spectral_norm_device(1e-10, cap);
            } else {
                std::vector<double> bh(q * n);
                ck(cudaMemcpyAsync(bh.data(), B.p, sizeof(double) * q * n, cudaMemcpyDeviceToHost,
                                   stream), "B to host");
                sync("B to host");
                b_spec = spectral_norm_host(bh, q, n, 1e-10, cap);
            }
            const double b2 = b_spec * b_spec;
            switch (cfg.alpha_rule) {
                case AXB_ALPHA_SAFE: alpha = 1.0 / b2; break;
                case AXB_ALPHA_PAPER:
                    alpha = 1.0 / b_spec;
                    alpha_outside = !(alpha < 2.0 / b2);
                    break;
                default:
                    alpha = cfg.alpha_value;
                    if (!(alpha > 0.0) || !(alpha < 2.0 / b2))
                        fail(AXB_CONFIG_ERROR, "fixed alpha %f outside (0, 2/‖B‖₂²)", alpha);
            }
        }

        // gram_ = gram_mmt(A) (solver.hpp:171): cached when it fits in HBM and the
        // run is long enough to repay it.  Forming G costs m_g·m·p FLOP on the DMMA
        // pipe (symmetric half, ~29 TFLOP/s); without it every iteration re-reads
        // the local A for g = A·A_iᵀ (8·m·p bytes at ~6.4 TB/s).  The horizon is the
        // solve's iteration budget (cfg.max_iter, the reference's 200000 by
        // default): a short fixed budget skips G, a long solve caches it.
        size_t free_b = 0, total_b = 0;
        ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
        const double gbytes = 8.0 * (double)m_g * (double)m;
        const double g_form_s = (double)m_g * (double)m * (double)p / (sharded ? 14.5e12 : 29e12);
        const double g_step_s = 8.0 * (double)m * (double)p / 6.4e12;
        const bool repays = (double)cfg.max_iter * g_step_s >= g_form_s;
        gram_cached = !sp_a && (opt.cache_gram == 1 ||
                                (opt.cache_gram < 0 && gbytes < 0.45 * (double)free_b &&
                                 gbytes <= 48e9 && repays));
        // one decision for all ranks: forming G gathers A (a collective), and a
        // rank whose free memory differed must not take the other branch
        if (sharded) gram_cached = global_sum(gram_cached ? 1.0 : 0.0) == (double)world;
        // association of the residual product (matrix-chain order): the reference
        // evaluates (A·X)·B, 2mpq + 2mqn FLOP; A·(X·B) costs 2pqn + 2mpn and is
        // taken when it is at least 5% cheaper (config 5: 3.96e13 vs 4.40e13;
        // never for a world-8 shard, whose m is m/8).  Same product to rounding.
        {
            const double left = (double)m * p * q + (double)m * q * n;
            const double right = (double)p * q * n + (double)m * p * n;
            const int e = env_int("AXB_CHAIN_XB", -1);
            chain_xb = !sp_a && !sp_b && (e >= 0 ? e != 0 : right < 0.95 * left);
        }
        T.alloc(std::max(m * q, chain_xb ? p * n : (uint64_t)0), "T");
        const int gparts = gemm_num_ctas((long long)m, (long long)std::max(n, m));
        gemm_sq.alloc(gparts, "gemm parts");
        gemm_diff.alloc(gparts, "gemm parts");
        if (gram_cached) {
            // G[:, local rows] = A_all · A_localᵀ (m_global × m); one GPU: G = A·Aᵀ
            G.alloc(m_g * m, "G");
            DevBuf<double> A_all;
            const double* Aa = A.p;
            if (sharded) {
                A_all.alloc(m_g * p, "A gathered");
                ck(cudaMemcpyAsync(A_all.p + row0 * p, A.p, sizeof(double) * m * p,
                                   cudaMemcpyDeviceToDevice, stream), "A slot");
                allgather_inplace(A_all.p, m * p);
                Aa = A_all.p;
            }
            GemmArgs ga{};
            ga.M = m_g; ga.N = m; ga.K = p;
            ga.A = Aa; ga.lda = p;
            ga.B = A.p; ga.ldb = p; ga.b_trans = 1;
            ga.D = G.p; ga.ldd = m;
            ga.store = 1;
            ga.sym = sharded ? 0 : 1;  // one GPU: G = A·Aᵀ symmetric, upper tiles + mirror
            launch_gemm(ga, stream);
            if (!sharded) launch_mirror_lower(G.p, (long long)m, (long long)m, stream);
            sync("G");  // A_all released at scope end
        } else {
            g.alloc(m, "g");
            // CSR A: g holds the scattered Gram row, exactly zero elsewhere
            if (sp_a) ck(cudaMemsetAsync(g.p, 0, sizeof(double) * m, stream), "g");
        }

        // r_ = C − (A·X0)·B (solver.hpp:173)
        ck(cudaStreamWaitEvent(stream, evRest, 0), "wait C, X0, X_ref");
        if (X0_in) {
            exact_residual_into(R.p, nullptr, nullptr, true);
        } else {
            ck(cudaMemcpyAsync(R.p, C.p, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, stream),
               "R = C");
        }
        c_fro = std::sqrt(global_sum(reduce_sumsq(C.p, m * n)));  // :179
        if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN) {   // :180-189
            ref_sq = reduce_sumsq(Xref.p, p * q);
            if (ref_sq == 0.0) fail(AXB_DOMAIN_ERROR, "solution_rrn: zero reference");
        }

        // iteration buffers and launch geometry
        y.alloc(q, "y");
        z.alloc(std::max<uint64_t>(n, n_loc * world), "z");
        P.m = (long long)m; P.p = (long long)p; P.q = (long long)q; P.n = (long long)n;
        P.row0 = (long long)row0;
        P.m_global = (long long)m_g;
        P.world = world;
        P.rank = rank;
        P.c0 = sharded ? std::min<long long>((long long)n, (long long)(rank * n_loc)) : 0;
        P.c1 = sharded ? std::min<long long>((long long)n, P.c0 + (long long)n_loc) : (long long)n;
        P.x0r = sharded ? std::min<long long>((long long)p, (long long)(rank * p_loc)) : 0;
        P.x1r = sharded ? std::min<long long>((long long)p, P.x0r + (long long)p_loc) : (long long)p;
        const int target = 148 * 4;
        P.r_tma = (n % 2 == 0) && opt_r_tma();
        if (P.r_tma) {
            // TMA ring: 2 CTAs per SM, rows split evenly, tiles of ≤2048 columns
            // (tunable for sweeps: AXB_R_CPS, AXB_R_STAGES, AXB_R_TILE)
            const int cps = env_int("AXB_R_CPS", 2);
            // few rows per CTA on wide rows (config 3: 28 rows of 8192 per CTA): two
            // 2048-column stages, same ring bytes, half the per-tile handshakes
            // (config 3 K2 0.1829 → 0.1818 ms, 3,785 → 3,824 it/s); many rows per CTA
            // (config 5: 221) keep four 1024-column stages (161.3 vs 160.9 it/s), and
            // so do rows longer than 16384 (config 5's world-8 shard, measured at the
            // copy roofline with 1024 × 4)
            const bool wide = m <= (uint64_t)64 * 148 * cps && n >= 4096 && n <= 16384;
            const int stages = env_int("AXB_R_STAGES", wide ? 2 : 4);
            const int tile = env_int("AXB_R_TILE", wide ? 2048 : 1024);
            P.r_grid = (int)std::min<uint64_t>((uint64_t)148 * cps, m);
            P.r_rows_per_cta = (int)((m + P.r_grid - 1) / P.r_grid);
            P.r_chunk = (int)std::min<uint64_t>(n, (uint64_t)tile);
            P.r_stages = std::max(2, std::min(stages, 16));
            P.r_zstage = env_int("AXB_R_ZSTAGE", 1);
            // rows per dynamic grab (tools/sweep_grab.sh): one row at a time.  With
            // 32-row grabs config 3's 8192 rows were 256 grabs over 296 CTAs (one
            // or two per SM, so some SMs streamed twice the rows of others), and
            // at config 5 the CTAs' concurrent rows sat 2 MB apart.  K2 time per
            // grab of 32 / 8 / 1 rows: config 3 0.189 / 0.193 / 0.183 ms, config 5
            // 5.37 / 5.25 / 5.16 ms.
            P.r_grab = std::max(1, std::min(32, env_int("AXB_R_GRAB", 1)));
        } else {
            int rgrid = (int)std::min<uint64_t>((uint64_t)target, std::max<uint64_t>(1, (m + 7) / 8));
            P.r_rows_per_cta = (int)((m + rgrid - 1) / rgrid);
            P.r_grid = (int)((m + P.r_rows_per_cta - 1) / P.r_rows_per_cta);
            P.r_chunk = (int)std::min<uint64_t>(n, 4096);
            if (P.r_chunk & 1) P.r_chunk += (n > (uint64_t)P.r_chunk) ? 1 : 0;
        }
        {
            auto rpc = [](uint64_t r) { return r >= 8 * 1184 ? 8 : r >= 4 * 1184 ? 4 : r >= 2 * 1184 ? 2 : 1; };
            // rows per CTA (1, 2, 4, 8; AXB_YG_RB overrides for the B rows): with
            // more than one, the shared vector is staged once per CTA and reused
            int rbq = rpc(q);
            if (const int e = env_int("AXB_YG_RB", 0); e == 1 || e == 2 || e == 4 || e == 8) rbq = e;
            P.yg_rbq = rbq;
            P.yg_rbm = rpc(m);
            const uint64_t blocks = (q + rbq - 1) / rbq + (gram_cached ? 0 : (m + P.yg_rbm - 1) / P.yg_rbm);
            P.yg_grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(1u << 20, blocks));
            if (const int e = env_int("AXB_YG_GRID", 0); e > 0) P.yg_grid = std::min(P.yg_grid, e);
            P.yg_pf = std::max(0, env_int("AXB_YG_PF", 0));
            // K4 as a TMA ring when K2 runs one (its ring geometry and carve-out) and
            // every streamed row is 16-byte aligned (B slice; A rows when g is formed)
            P.yg_tma = (P.r_tma && P.c1 > P.c0 && ((P.c1 - P.c0) % 2 == 0) && (P.c0 % 2 == 0) &&
                        (gram_cached || p % 2 == 0) && env_int("AXB_YG_TMA", 1)) ? 1 : 0;
            P.sel_early = env_int("AXB_SEL_EARLY", 0);
        }
        // small systems run one persistent kernel per batch (decided below; the
        // z row chunks depend on it)
        const double persist_ws = 8.0 * ((double)m * n + (double)q * n + 2.0 * p * q + (double)m * p);
        const int persist_force = env_int("AXB_PERSIST", -1);
        // CSR operands always take the persistent general body (its phases iterate
        // stored entries); their working set is the touched rows, not m·n
        const bool persist_path =
            !sharded && (sp_a || sp_b || persist_force == 1 || (persist_force < 0 && persist_ws <= 64e6));
        {
            // K4b+K5 in small units over several waves, so the tail evens out:
            // X one row per warp (8 rows per CTA), z slabs of 512 columns ×
            // chunks of AXB_Z_JROWS rows of the B slice: 128 for the graph path
            // (k_zx), 32 in the persistent general body, whose z items are few and
            // each a chain of dependent L2 round trips (config 2: 29.2k → 35.6k it/s)
            const long long xrows = P.x1r - P.x0r;
            P.x_ctas = (int)std::max<long long>(1, (xrows + kZxWarps - 1) / kZxWarps);
            P.z_nslab = (int)std::max<long long>(1, (P.c1 - P.c0 + 511) / 512);
            const long long jr = std::max(1, env_int("AXB_Z_JROWS", persist_path ? 32 : 128));
            P.z_jrows = (int)std::min<long long>((long long)q, jr);
            P.z_nj = (int)((q + P.z_jrows - 1) / P.z_jrows);
        }
        zpart.alloc((size_t)P.z_nj * n, "zpart");
        zcnt.alloc(P.z_nslab, "zcnt");
        ck(cudaMemsetAsync(zcnt.p, 0, sizeof(unsigned) * P.z_nslab, stream), "zcnt");
        xpart.alloc(std::max<size_t>(2 * 1184, (size_t)P.x_ctas), "xpart");
        // per-CTA records of K2 (r_grid CTAs) and of the persistent general body (≤ one
        // CTA per SM, whatever m is)
        rrec.alloc(std::max<size_t>((size_t)P.r_grid, 1024), "rrec");
        tr_row.alloc(trace_cap, "trace");
        forced.alloc(trace_cap, "forced rows");
        gsum.alloc(((sharded ? m_g : m) + 31) / 32, "group sums");
        tr_metric.alloc(trace_cap, "trace");
        tr_rel.alloc(trace_cap, "trace");
        flags.alloc(m, "flags");
        st.alloc(1, "state");

        P.A = A.p; P.B = B.p; P.R = R.p; P.X = X.p; P.Xref = Xref.p;
        P.a_sq = a_sq.p; P.rbk_cum = rbk_cum.p;
        P.r_sq = sharded ? r_sq.p + row0 : r_sq.p;
        P.r_sq_g = sharded ? r_sq.p : nullptr;
        P.G = gram_cached ? G.p : nullptr;
        P.g = g.p; P.y = y.p; P.z = z.p; P.zpart = zpart.p; P.zcnt = zcnt.p; P.xpart = xpart.p;
        P.rrec = rrec.p; P.trace_row = tr_row.p; P.trace_metric = tr_metric.p;
        P.trace_rel = tr_rel.p; P.trace_cap = trace_cap; P.member_flags = flags.p; P.st = st.p;
        P.forced_rows = forced.p;
        P.gsum = gsum.p;
        P.pack = sharded ? pack.p : nullptr;
        P.pack_send = pack_send.p;
        P.recs = recs.p;
        P.a_sq_g = sharded ? a_sq_g.p : a_sq.p;
        P.alpha = alpha;
        P.theta = cfg.method == AXB_RGRBK ? cfg.theta : 0.5;
        P.a_fro_sq = a_fro_sq;
        P.tol = cfg.tol;
        P.ref_sq = ref_sq > 0.0 ? ref_sq : 1.0;
        P.c_fro = c_fro;
        P.method = cfg.method;
        P.stop_kind = cfg.stop_kind;
        // sharded too: every rank sees all of r_sq; 2 = always walk (test hook)
        P.tie_guard = opt.tie_guard == 2 ? 2 : (opt.tie_guard ? 1 : 0);
        {
            // greedy pre-selection spread over the SMs (k_sel_greedy) once the
            // O(m) membership pass outweighs one more PDL-chained launch
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt.device);
            const long long ng = (long long)(m + 31) / 32;
            const bool greedy = cfg.method == AXB_GRBK || cfg.method == AXB_RGRBK;
            P.sel_split = (!sharded && greedy && env_int("AXB_SEL_SPLIT", ng >= 64 ? 1 : 0)) ? 1 : 0;
            P.sel_grid = (int)std::max<long long>(1, std::min<long long>(sms, (ng + 3) / 4));
            // sharded: k_sel1's membership pass and k_pack's row copy across the SMs
            P.sel1_grid = greedy ? P.sel_grid : 1;
            P.pack_grid = (int)std::max<long long>(
                1, std::min<long long>(sms, (long long)(n + p + 2 + 1023) / 1024));
        }
        // small systems (per-iteration working set L2-resident): one persistent
        // cooperative kernel per batch instead of a graph of 3 kernels/iteration
        {
            int sms = 148;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, opt.device);
            if (opt.sm_share > 0) sms = std::min(sms, (int)opt.sm_share);
            P.persist = persist_path;
            // grid: enough SMs for the L2 bandwidth of R, few enough for cheap grid syncs
            const int want = (int)std::min<double>(sms, std::max(64.0, (double)m * n / 16384.0));
            P.persist_grid = env_int("AXB_PERSIST_GRID", want);
            // latency body (selection state in shared memory, z = BᵀB·R_iᵀ, two grid
            // barriers per iteration) when BᵀB is small enough to cache: tiny
            // systems such as config 1.  AXB_PERSIST_LAT = threads per CTA (256 or
            // 128), 0 = off; AXB_PERSIST_BTB = 1 forces it for larger n.
            const int lat_env = env_int("AXB_PERSIST_LAT", 256);
            const int bforce = env_int("AXB_PERSIST_BTB", -1);
            const bool btb_ok = bforce == 1 || (bforce < 0 && 8.0 * (double)n * (double)n <= 16e6);
            P.persist_lat = (P.persist && (long long)m <= kPersistLatRows && lat_env != 0 &&
                             (btb_ok || sp_b))
                                ? (lat_env == 128 ? 128 : 256) : 0;
            // latency-bound: every SM's load parallelism, barrier cost barely grows
            if (P.persist_lat) P.persist_grid = env_int("AXB_PERSIST_GRID", sms);
        }
        // z = BᵀB·R_iᵀ in the latency body (btb_, solver.hpp:172, :293): y and z
        // then share one phase; cached when BᵀB is small (L2-resident)
        P.BtB = nullptr;
        if (P.persist_lat && !sp_b) {  // CSR B: the latency body reads the CSR BᵀB
            {
                BtB.alloc(n * n, "BtB");
                DevBuf<double> Bt;
                Bt.alloc(q * n, "B transposed");
                launch_transpose(B.p, (long long)q, (long long)n, Bt.p, stream);
                GemmArgs ga{};
                ga.M = n; ga.N = n; ga.K = q;
                ga.A = Bt.p; ga.lda = q;
                ga.B = Bt.p; ga.ldb = q; ga.b_trans = 1;
                ga.D = BtB.p; ga.ldd = n;
                ga.store = 1;
                ga.sym = 1;
                launch_gemm(ga, stream);
                launch_mirror_lower(BtB.p, (long long)n, (long long)n, stream);
                sync("BtB");  // Bt released at scope end
                P.BtB = BtB.p;
            }
        }
        P.vec2 = (n % 2) == 0;
        P.a_rp = sp_a ? a_rp.p : nullptr; P.a_ci = a_ci.p; P.a_v = a_v.p;
        P.g_rp = sp_a ? g_rp.p : nullptr; P.g_ci = g_ci.p; P.g_v = g_v.p;
        P.b_rp = sp_b ? b_rp.p : nullptr; P.b_ci = b_ci.p; P.b_v = b_v.p;
        P.bt_rp = sp_b ? bt_rp.p : nullptr; P.bt_ci = bt_ci.p; P.bt_v = bt_v.p;
        P.btb_rp = sp_b ? btb_rp.p : nullptr; P.btb_ci = btb_ci.p; P.btb_v = btb_v.p;

        // DevState: RngStream(cfg.seed) (rng.hpp:20-25), k = 0
        DevState s0{};
        uint64_t x = cfg.seed;
        for (int i = 0; i < 4; ++i) {
            x += 0x9e3779b97f4a7c15ULL;
            uint64_t zz = x;
            zz = (zz ^ (zz >> 30)) * 0xbf58476d1ce4e5b9ULL;
            zz = (zz ^ (zz >> 27)) * 0x94d049bb133111ebULL;
            s0.rng[i] = zz ^ (zz >> 31);
        }
        if (!s0.rng[0] && !s0.rng[1] && !s0.rng[2] && !s0.rng[3]) s0.rng[0] = 1;
        s0.status = ST_RUN;
        s0.fin_mode = FIN_ITERATION;
        s0.argmax = -1;
        *hs = s0;
        ck(cudaMemcpyAsync(st.p, hs, sizeof(DevState), cudaMemcpyHostToDevice, stream), "state");
        adopt_norms();
        if (sharded) {
            // every collective of the iteration once, eagerly: NCCL sets up its
            // connections lazily at a collective's first call, which must not
            // happen inside a graph capture (a first steps(k ≥ graph_iters) call
            // captures at once).  y and z are recomputed before any use.
            allreduce(y.p, y.p, q);
            allgather_inplace(z.p, n_loc);
            allreduce(pack_send.p, pack.p, n + p + 2);
        }
        sync("init");
        pull_state();
    }

    // ‖B‖₂ on the device: the reference's power iteration (decomp.hpp:207-239: same
    // start vector, same stop test) applied to the small Gram M = B·Bᵀ (q ≤ n) or
    // BᵀB, formed once by the DMMA GEMM and then L2-resident; the stop test runs
    // on the device and the host looks every 32 iterations.
    double spectral_norm_device(double tol, size_t max_iter) {
        if (reduce_sumsq(B.p, q * n) == 0.0) fail(AXB_DOMAIN_ERROR, "spectral_norm: zero matrix");
        const bool use_mtm = n <= q;
        const size_t dim = use_mtm ? n : q;
        if (8.0 * (double)dim * (double)dim > 16e9) return spectral_norm_device_2pass(tol, max_iter);
        DevBuf<double> M, Bt, v, w, ps;
        M.alloc(dim * dim, "power Gram");
        GemmArgs ga{};
        ga.M = dim; ga.N = dim; ga.store = 1; ga.b_trans = 1;
        if (use_mtm) {  // M = BᵀB = (Bᵀ)(Bᵀ)ᵀ
            Bt.alloc(q * n, "B transposed");
            launch_transpose(B.p, (long long)q, (long long)n, Bt.p, stream);
            ga.K = q; ga.A = Bt.p; ga.lda = q; ga.B = Bt.p; ga.ldb = q;
        } else {        // M = B·Bᵀ
            ga.K = n; ga.A = B.p; ga.lda = n; ga.B = B.p; ga.ldb = n;
        }
        ga.D = M.p; ga.ldd = dim;
        ga.sym = 1;
        launch_gemm(ga, stream);
        launch_mirror_lower(M.p, (long long)dim, (long long)dim, stream);
        std::vector<double> v0 = power_start(dim);
        v.alloc(dim, "power v");
        w.alloc(dim, "power w");
        ps.alloc(4, "power state");
        ck(cudaMemcpyAsync(v.p, v0.data(), sizeof(double) * dim, cudaMemcpyHostToDevice, stream),
           "v0");
        ck(cudaMemsetAsync(ps.p, 0, sizeof(double) * 4, stream), "power state");
        double h[4] = {0, 0, 0, 0};
        for (size_t done = 0; done < max_iter; done += 32) {
            for (int i = 0; i < 32; ++i) {
                launch_rowdot(M.p, (long long)dim, (long long)dim, v.p, w.p, stream);
                launch_power_step2(v.p, w.p, (long long)dim, ps.p, tol, (double)max_iter, stream);
            }
            ck(cudaMemcpyAsync(h, ps.p, sizeof h, cudaMemcpyDeviceToHost, stream), "power");
            sync("power");
            if (h[3] != 0.0) break;
        }
        if (h[3] == 1.0) return h[1];
        AxbError e{AXB_CONVERGENCE_ERROR, "spectral_norm: power iteration did not converge"};
        e.val = std::sqrt(std::abs(h[0]));
        throw e;
    }

    // two GEMV passes over B per iteration (for a Gram too large to form)
    double spectral_norm_device_2pass(double tol, size_t max_iter) {
        const bool use_mtm = n <= q;
        const size_t dim = use_mtm ? n : q, other = use_mtm ? q : n;
        std::vector<double> v0 = power_start(dim);
        DevBuf<double> v, vn, w, t, part, out2;
        DevBuf<unsigned int> cnt;
        v.alloc(dim, "power v");
        vn.alloc(dim, "power v");
        w.alloc(dim, "power w");
        t.alloc(other, "power t");
        out2.alloc(2, "power out");
        const int nslab = (int)((n + 255) / 256);
        const int nj = (int)std::max<size_t>(1, std::min<size_t>((592 + nslab - 1) / nslab, (q + 7) / 8));
        const int jrows = (int)((q + nj - 1) / nj);
        const int nj2 = (int)((q + jrows - 1) / jrows);
        part.alloc((size_t)nj2 * n, "power part");
        cnt.alloc(nslab, "power cnt");
        ck(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned) * nslab, stream), "cnt");
        ck(cudaMemcpyAsync(v.p, v0.data(), sizeof(double) * dim, cudaMemcpyHostToDevice, stream),
           "v0");
        double lambda = 0.0, h2[2];
        for (size_t it = 0; it < max_iter; ++it) {
            if (use_mtm) {  // w = Bᵀ(B v)
                launch_rowdot(B.p, (long long)q, (long long)n, v.p, t.p, stream);
                launch_coldot(B.p, (long long)q, (long long)n, t.p, w.p, part.p, cnt.p, nj2, jrows,
                              stream);
            } else {        // w = B(Bᵀ v)
                launch_coldot(B.p, (long long)q, (long long)n, v.p, t.p, part.p, cnt.p, nj2, jrows,
                              stream);
                launch_rowdot(B.p, (long long)q, (long long)n, t.p, w.p, stream);
            }
            launch_power_step(v.p, w.p, vn.p, (long long)dim, out2.p, stream);
            ck(cudaMemcpyAsync(h2, out2.p, sizeof h2, cudaMemcpyDeviceToHost, stream), "power");
            sync("power");
            const double rayleigh = h2[0], wn = h2[1];
            if (wn == 0.0) return 0.0;
            std::swap(v.p, vn.p);
            if (it > 0 && std::abs(rayleigh - lambda) <= 0.5 * tol * std::abs(rayleigh))
                return std::sqrt(rayleigh);
            lambda = rayleigh;
        }
        AxbError e{AXB_CONVERGENCE_ERROR, "spectral_norm: power iteration did not converge"};
        e.val = std::sqrt(std::abs(lambda));
        throw e;
    }

    // D = C − (A·X)·B into out (store) with optional Σ D² and Σ (Rold − D)² partials
    void exact_residual_into(double* out, double* sq, const double* rold, bool store) {
        if (chain_xb) {  // T = X·B (p×n), then C − A·T
            GemmArgs t1{};
            t1.M = p; t1.N = n; t1.K = q;
            t1.A = X.p; t1.lda = q;
            t1.B = B.p; t1.ldb = n;
            t1.D = T.p; t1.ldd = n;
            t1.store = 1;
            launch_gemm(t1, stream);
            GemmArgs t2{};
            t2.M = m; t2.N = n; t2.K = p;
            t2.A = A.p; t2.lda = p;
            t2.B = T.p; t2.ldb = n;
            t2.D = out; t2.ldd = n;
            t2.Cin = C.p; t2.ldc = n;
            t2.Rold = rold; t2.ldr = n;
            t2.sq_part = sq;
            t2.diff_part = rold ? gemm_diff.p : nullptr;
            t2.store = store ? 1 : 0;
            launch_gemm(t2, stream);
            return;
        }
        if (sp_a) {  // T = A·X over A's stored entries (matrix.hpp sparse matmul)
            launch_spmm_csr(a_rp.p, a_ci.p, a_v.p, (long long)m, X.p, (long long)q, T.p, stream);
        } else {
            GemmArgs t1{};
            t1.M = m; t1.N = q; t1.K = p;
            t1.A = A.p; t1.lda = p;
            t1.B = X.p; t1.ldb = q;
            t1.D = T.p; t1.ldd = q;
            t1.store = 1;
            launch_gemm(t1, stream);
        }
        GemmArgs t2{};
        t2.M = m; t2.N = n; t2.K = q;
        t2.A = T.p; t2.lda = q;
        t2.B = B.p; t2.ldb = n;
        t2.D = out; t2.ldd = n;
        t2.Cin = C.p; t2.ldc = n;
        t2.Rold = rold; t2.ldr = n;
        t2.sq_part = sq;
        t2.diff_part = rold ? gemm_diff.p : nullptr;
        t2.store = store ? 1 : 0;
        launch_gemm(t2, stream);
    }

    // r_sq_, r_fro_sq_, reductions of the current R (solver.hpp:174-177, :468-476)
    void adopt_norms() {
        if (sharded) {
            // local ‖X−X_ref‖² first: this shard's record carries it
            if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN) launch_err_fresh(P, stream);
            launch_r(P, stream, false);
            gather_norms();
            launch_sel1(P, stream, 0);
        } else {
            launch_r(P, stream, false);
            if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN) launch_err_fresh(P, stream);
        }
        sel_valid = false;
    }

    // ---------------------------------------------------------------- selection
    void rollback() {
        launch_rollback(P, stream);
        sel_valid = false;
    }

    void ensure_selection() {
        if (!sel_valid && sharded) {
            launch_sel1(P, stream, 2);  // k_sel1 (select only) + k_pack
            allreduce(pack_send.p, pack.p, n + p + 2);
            kernel_launches += 2;
            sel_valid = true;
        } else if (!sel_valid) {
            launch_select(P, stream, cfg.method, P.theta, 0);
            ++kernel_launches;
            sel_valid = true;  // confirmed (or error) at the next state pull
        }
    }

    // ---------------------------------------------------------------- iteration
    // one iteration; sharded: y partial → allreduce, z slice → allgather, local R
    // update → ONE grouped allgather (‖R_l‖² slices + shard records) → global stop
    // logic and the selection over the global rows, identical on every rank →
    // owner pack → row allreduce: 4 collectives, 5 kernels

    void enqueue_iteration() {
        launch_yg(P, stream, !gram_cached);
        if (sharded) allreduce(y.p, y.p, q);
        launch_zx(P, stream);
        if (sharded) allgather_inplace(z.p, n_loc);
        launch_r(P, stream, true);
        if (P.sel_split) launch_sel_greedy(P, stream);
        if (sharded) {
            gather_norms();
            launch_sel1(P, stream, 1);
            allreduce(pack_send.p, pack.p, n + p + 2);
        }
    }
    int launches_per_iteration() const { return sharded ? 5 : (P.sel_split ? 4 : 3); }
    void launch_iteration() {
        enqueue_iteration();
        kernel_launches += launches_per_iteration();
    }

    void build_graph() {
        cudaGraph_t g0 = nullptr;
        ck(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal), "capture");
        for (int i = 0; i < graph_iters; ++i) enqueue_iteration();
        ck(cudaStreamEndCapture(stream, &g0), "capture end");
        ck(cudaGraphInstantiate(&graph, g0, 0), "graph instantiate");
        cudaGraphDestroy(g0);
    }

    // runs up to nb iterations from the current k; returns iterations executed
    uint64_t batch(uint64_t nb, int run_mode) {
        batch_launch(nb, run_mode, false);
        return batch_collect();
    }
    // a persistent-kernel handle whose kernel a multi-system launch runs
    // (axb_solvers_run): only the control block is armed here
    // CSR operands run only on the persistent body (per-kernel profiling is the
    // dense graph path's measurement hook)
    bool use_persist() const { return P.persist && (!profiling || sp_a || sp_b); }
    bool batchable() const { return use_persist(); }
    void batch_launch(uint64_t nb, int run_mode, bool external) {
        launch_ctrl(st.p, k, k + nb, FIN_ITERATION, run_mode, 0, stream);
        ++kernel_launches;
        if (external) {
            ++kernel_launches;  // the shared k_persist_batch launch
            return;
        }
        if (use_persist()) {
            // the kernel selects at the top of each iteration itself
            const int e = launch_persist(P, stream);
            if (e != 0) ck(static_cast<cudaError_t>(e), "persistent kernel launch");
            ++kernel_launches;
        } else {
            ensure_selection();
        }
        if (use_persist()) {
            // nothing more to enqueue
        } else if (profiling) {
            // 9 events per iteration around every op: [y][y allreduce][z, X][z allgather]
            // [R update (+ K3)][r_sq/record allgather][selection + pack][row allreduce]
            if (prof_ev.size() < kProfEv * nb) {
                size_t have = prof_ev.size();
                prof_ev.resize(kProfEv * nb);
                for (size_t i = have; i < prof_ev.size(); ++i) ck(cudaEventCreate(&prof_ev[i]), "ev");
            }
            for (uint64_t i = 0; i < nb; ++i) {
                cudaEvent_t* e = &prof_ev[kProfEv * i];
                ck(cudaEventRecord(e[0], stream), "ev");
                launch_yg(P, stream, !gram_cached);
                ck(cudaEventRecord(e[1], stream), "ev");
                if (sharded) allreduce(y.p, y.p, q);
                ck(cudaEventRecord(e[2], stream), "ev");
                launch_zx(P, stream);
                ck(cudaEventRecord(e[3], stream), "ev");
                if (sharded) allgather_inplace(z.p, n_loc);
                ck(cudaEventRecord(e[4], stream), "ev");
                launch_r(P, stream, true);
                if (P.sel_split) launch_sel_greedy(P, stream);  // timed with K2: its tail
                ck(cudaEventRecord(e[5], stream), "ev");
                if (sharded) gather_norms();
                ck(cudaEventRecord(e[6], stream), "ev");
                if (sharded) launch_sel1(P, stream, 1);
                ck(cudaEventRecord(e[7], stream), "ev");
                if (sharded) allreduce(pack_send.p, pack.p, n + p + 2);
                ck(cudaEventRecord(e[8], stream), "ev");
                kernel_launches += launches_per_iteration();
            }
        } else if (nb < (uint64_t)graph_iters || emulated) {
            for (uint64_t i = 0; i < nb; ++i) launch_iteration();
        } else {
            if (!graph) build_graph();
            const uint64_t launches = (nb + graph_iters - 1) / graph_iters;
            for (uint64_t i = 0; i < launches; ++i) ck(cudaGraphLaunch(graph, stream), "graph launch");
            kernel_launches += (uint64_t)launches_per_iteration() * nb;
        }
        last_nb = nb;
    }
    uint64_t batch_collect() {
        const uint64_t nb = last_nb;
        (void)nb;
        pull_state();
        if (profiling) {
            const uint64_t done = hs->k - k;
            for (uint64_t i = 0; i < done; ++i) {
                const cudaEvent_t* e = &prof_ev[kProfEv * i];
                float t[kProfEv - 1];
                for (int j = 0; j + 1 < kProfEv; ++j)
                    ck(cudaEventElapsedTime(&t[j], e[j], e[j + 1]), "elapsed");
                yg_ms += t[0];
                coll_ms[0] += t[1];
                zx_ms += t[2];
                coll_ms[1] += t[3];
                k2_ms += t[4];
                coll_ms[2] += t[5];
                sel_ms += t[6];
                coll_ms[3] += t[7];
                ++k2_launches;
            }
        }
        sel_valid = hs->sel_valid != 0;
        const uint64_t done = hs->k - k;
        if (done) {
            ck(cudaMemcpyAsync(h_trace_row, tr_row.p, sizeof(long long) * done,
                               cudaMemcpyDeviceToHost, stream), "trace");
            ck(cudaMemcpyAsync(h_trace_metric, tr_metric.p, sizeof(double) * done,
                               cudaMemcpyDeviceToHost, stream), "trace");
            ck(cudaMemcpyAsync(h_trace_rel, tr_rel.p, sizeof(double) * done,
                               cudaMemcpyDeviceToHost, stream), "trace");
            sync("trace");
        }
        k = hs->k;
        if (hs->status == ST_ERROR) raise_state();
        return done;
    }

    void reset_status() { launch_ctrl(st.p, k, k, FIN_ITERATION, 0, 1, stream); }

    // k step() calls (acceptance.cpp:128-141), optional run()-style refresh
    void steps(uint64_t count, uint64_t* rows, bool mirror_refresh) {
        reset_status();
        uint64_t got = 0;
        cudaEventRecord(ev0, stream);
        while (got < count) {
            uint64_t nb = std::min<uint64_t>(count - got, trace_cap);
            const uint64_t ri = cfg.refresh_interval;
            if (mirror_refresh && ri > 0) nb = std::min<uint64_t>(nb, ri - k % ri);
            const uint64_t done = batch(nb, 0);
            if (rows)
                for (uint64_t t = 0; t < done; ++t) rows[got + t] = (uint64_t)h_trace_row[t];
            got += done;
            if (done != nb) fail(AXB_CUDA_ERROR, "batch stopped early (%llu of %llu)",
                                 (unsigned long long)done, (unsigned long long)nb);
            if (mirror_refresh && ri > 0 && k % ri == 0) checkpoint();
        }
        cudaEventRecord(ev1, stream);
        sync("steps");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        loop_ms = ms;
    }

    // k iterations on a given index stream (the reference's), e.g. to replay a
    // randomized run: X, R and the metrics follow exactly as step() would
    void replay(uint64_t count, const uint64_t* rows_in, bool mirror_refresh) {
        reset_status();
        rollback();
        launch_set_replay(st.p, 1, stream);
        std::vector<long long> chunk(trace_cap);
        uint64_t got = 0;
        cudaEventRecord(ev0, stream);
        try {
            while (got < count) {
                uint64_t nb = std::min<uint64_t>(count - got, trace_cap);
                const uint64_t ri = cfg.refresh_interval;
                if (mirror_refresh && ri > 0) nb = std::min<uint64_t>(nb, ri - k % ri);
                for (uint64_t t = 0; t < nb; ++t) chunk[t] = (long long)rows_in[got + t];
                ck(cudaMemcpyAsync(forced.p, chunk.data(), sizeof(long long) * nb,
                                   cudaMemcpyHostToDevice, stream), "forced rows");
                sel_valid = false;  // the first selection of the batch reads slot 0
                const uint64_t done = batch(nb, 0);
                got += done;
                if (done != nb) fail(AXB_CUDA_ERROR, "replay stopped early");
                if (mirror_refresh && ri > 0 && k % ri == 0) checkpoint();
                sync("replay chunk");  // chunk buffer reuse
            }
        } catch (...) {
            launch_set_replay(st.p, 0, stream);
            sel_valid = false;
            throw;
        }
        cudaEventRecord(ev1, stream);
        launch_set_replay(st.p, 0, stream);
        sel_valid = false;
        sync("replay");
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        loop_ms = ms;
    }

    void not_sharded(const char* what) {
        if (sharded)
            fail(AXB_CONFIG_ERROR, "%s is not available on a row-sharded solver (use step/steps/"
                                   "replay/run)", what);
    }
    void set_err_sq(double v) {  // publish a host-reduced ‖X−X_ref‖² into DevState
        ck(cudaMemcpyAsync(reinterpret_cast<char*>(st.p) + offsetof(DevState, err_sq), &v,
                           sizeof(double), cudaMemcpyHostToDevice, stream), "err_sq");
        sync("err_sq");
    }

    void update_row(uint64_t i) {  // solver.hpp:264-318
        not_sharded("update_row");
        if (i >= m) fail(AXB_SHAPE_ERROR, "update_row: row %llu out of range", (unsigned long long)i);
        if (!(a_sq_h[i] > 0.0)) fail(AXB_DOMAIN_ERROR, "update_row: zero row selected");
        rollback();
        launch_set_sel(st.p, (long long)i, alpha / a_sq_h[i], stream);
        launch_ctrl(st.p, k, k + 1, FIN_UPDATE_ROW, 0, 1, stream);
        if (sp_a || sp_b) {  // one pass of the persistent body on the given row
            const int e = launch_persist(P, stream);
            if (e != 0) ck(static_cast<cudaError_t>(e), "persistent kernel launch");
            ++kernel_launches;
        } else {
            launch_iteration();
        }
        launch_ctrl(st.p, k, k, FIN_ITERATION, 0, 0, stream);
        pull_state();
        sel_valid = false;
        if (hs->status == ST_ERROR) raise_state();
    }

    // ---------------------------------------------------------------- metrics
    double current_metric() {
        pull_state();
        if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN) return hs->err_sq / ref_sq;
        return current_residual_rel();
    }
    double current_residual_rel() {
        pull_state();
        const double s = hs->r_fro_sq;
        return std::sqrt(std::max(s, 0.0)) / (c_fro > 0.0 ? c_fro : 1.0);
    }
    double exact_residual_rel() {  // solver.hpp:417-419
        gather_X();
        exact_residual_into(nullptr, gemm_sq.p, nullptr, false);
        launch_reduce_parts(gemm_sq.p, gemm_num_ctas((long long)m, (long long)n), scal.p, stream);
        double s = 0.0;
        ck(cudaMemcpyAsync(&s, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream), "exact");
        sync("exact residual");
        s = global_sum(s);
        return std::sqrt(s) / (c_fro > 0.0 ? c_fro : 1.0);
    }
    double exact_metric() {  // solver.hpp:412-416
        if (cfg.stop_kind == AXB_STOP_SOLUTION_RRN) {
            launch_err_fresh(P, stream);
            pull_state();
            if (!sharded) return hs->err_sq / ref_sq;
            const double e = global_sum(hs->err_sq);
            set_err_sq(e);
            return e / ref_sq;
        }
        return exact_residual_rel();
    }
    double residual_drift() {  // solver.hpp:423
        gather_X();
        exact_residual_into(nullptr, nullptr, R.p, false);
        launch_reduce_parts(gemm_diff.p, gemm_num_ctas((long long)m, (long long)n), scal.p, stream);
        double s = 0.0;
        ck(cudaMemcpyAsync(&s, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream), "drift");
        sync("drift");
        return std::sqrt(global_sum(s));
    }
    void checkpoint() {  // solver.hpp:427-436
        launch_err_fresh(P, stream);
        pull_state();
        const bool finite = global_sum(hs->x_finite ? 0.0 : 1.0) == 0.0;
        if (!finite) {
            AxbError e{AXB_DIVERGENCE_ERROR, ""};
            e.k = k;
            e.val = std::sqrt(std::max(hs->r_fro_sq, 0.0));
            char buf[160];
            snprintf(buf, sizeof buf, "divergence at iteration %llu, residual frobenius norm %f",
                     (unsigned long long)k, e.val);
            e.msg = buf;
            throw e;
        }
        rollback();
        gather_X();
        // exact residual written in place over R; the epilogue reads R_old first
        exact_residual_into(R.p, nullptr, R.p, true);
        launch_reduce_parts(gemm_diff.p, gemm_num_ctas((long long)m, (long long)n), scal.p, stream);
        double d2 = 0.0;
        ck(cudaMemcpyAsync(&d2, scal.p, sizeof(double), cudaMemcpyDeviceToHost, stream), "drift");
        sync("checkpoint drift");
        d2 = global_sum(d2);
        adopt_norms();
        sync("checkpoint");
        const double drift = std::sqrt(d2);
        if (drift > 1e-8 * (1.0 + c_fro))
            fail(AXB_INVARIANT_ERROR, "residual drift guard tripped at iteration %llu",
                 (unsigned long long)k);
    }
    void resync() {  // solver.hpp:478
        rollback();
        gather_X();
        exact_residual_into(R.p, nullptr, nullptr, true);
        adopt_norms();
    }

    // ---------------------------------------------------------------- run()
    // run() (solver.hpp:337-372) as a resumable state machine, so that
    // axb_solvers_run can advance many handles through one batched launch
    struct RunCtx {
        axb_report* rep = nullptr;
        uint64_t *trace_k = nullptr, *trace_row = nullptr;
        double *trace_rrn = nullptr, *trace_rel = nullptr, *x_out = nullptr;
        uint64_t trace_cap_out = 0, ntrace = 0, k_before = 0, nb = 0;
        bool converged = false, done = false;
        std::chrono::steady_clock::time_point t0;
    };
    void run_begin(RunCtx& c) {
        std::memset(c.rep, 0, sizeof *c.rep);
        c.rep->alpha = alpha;
        c.rep->seed = cfg.seed;
        c.rep->alpha_outside_bound = alpha_outside;
        reset_status();
        c.ntrace = 0;
        c.converged = exact_metric() <= cfg.tol;  // :344
        c.t0 = std::chrono::steady_clock::now();
        cudaEventRecord(ev0, stream);
        c.done = c.converged || k >= cfg.max_iter;
    }
    // next segment length, or false when the loop ends here (:346-347)
    bool run_segment(RunCtx& c) {
        if (c.done) return false;
        pull_state();
        if (!(hs->r_fro_sq > 0.0)) {  // :347
            c.done = true;
            return false;
        }
        uint64_t nb = std::min<uint64_t>(cfg.max_iter - k, trace_cap);
        const uint64_t ri = cfg.refresh_interval;
        if (ri > 0) nb = std::min<uint64_t>(nb, ri - k % ri);
        c.k_before = k;
        c.nb = nb;
        return true;
    }
    void run_after(RunCtx& c, uint64_t done) {
        if (cfg.record_trace) {
            for (uint64_t t = 0; t < done; ++t) {
                const uint64_t kk = c.k_before + t;
                if (!trace_point_due(kk)) continue;  // :349-350
                if (c.ntrace < c.trace_cap_out) {
                    if (c.trace_k) c.trace_k[c.ntrace] = kk;
                    if (c.trace_rrn) c.trace_rrn[c.ntrace] = h_trace_metric[t];
                    if (c.trace_rel) c.trace_rel[c.ntrace] = h_trace_rel[t];
                    if (c.trace_row) c.trace_row[c.ntrace] = (uint64_t)h_trace_row[t];
                }
                ++c.ntrace;
            }
        }
        const uint64_t ri = cfg.refresh_interval;
        if (hs->status == ST_ZERO) {
            launch_ctrl(st.p, k, k, FIN_ITERATION, 0, 1, stream);
            c.done = true;
            return;
        }
        if (hs->status == ST_PAUSE) {  // :351-358
            launch_ctrl(st.p, k, k, FIN_ITERATION, 1, 1, stream);
            if (exact_metric() <= cfg.tol) c.converged = true;
            else resync();
        }
        if (!c.converged && ri > 0 && k % ri == 0) checkpoint();  // :359-360
        c.done = c.converged || k >= cfg.max_iter;
    }
    void run_fail(RunCtx& c, const AxbError& e) {
        c.rep->iterations = k;
        c.rep->diverged_iteration = e.k;
        c.rep->diverged_residual = e.val;
        c.done = true;
    }
    void run_end(RunCtx& c) {
        cudaEventRecord(ev1, stream);
        sync("run");
        const auto t1 = std::chrono::steady_clock::now();
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        loop_ms = ms;
        axb_report* rep = c.rep;
        rep->iterations = k;
        rep->wall_seconds = std::chrono::duration<double>(t1 - c.t0).count();
        rep->terminated_by = c.converged ? AXB_TERMINATED_TOLERANCE : AXB_TERMINATED_MAX_ITER;
        rep->final_rrn = exact_metric();
        rep->final_residual_rel = exact_residual_rel();
        pull_state();
        rep->skipped_zero_rows = hs->skipped_zero_rows;
        rep->trace_len = c.ntrace;
        if (c.x_out) {
            gather_X();
            sync("X gather");
            d2h_copy(c.x_out, X.p, sizeof(double) * p * q, stream);
        }
    }
    void run(axb_report* rep, uint64_t* trace_k, double* trace_rrn, double* trace_rel,
             uint64_t* trace_row, uint64_t trace_cap_out, double* x_out) {
        RunCtx c;
        c.rep = rep;
        c.trace_k = trace_k;
        c.trace_rrn = trace_rrn;
        c.trace_rel = trace_rel;
        c.trace_row = trace_row;
        c.trace_cap_out = trace_cap_out;
        c.x_out = x_out;
        run_begin(c);
        try {
            while (run_segment(c)) run_after(c, batch(c.nb, 1));
        } catch (AxbError& e) {
            run_fail(c, e);
            throw;
        }
        run_end(c);
    }

    // ---------------------------------------------------------------- public selects
    uint64_t select_consume(int method, double theta) {
        not_sharded("select_*");
        rollback();
        reset_status();
        launch_select(P, stream, method, theta, 1);
        pull_state();
        if (hs->status == ST_ERROR) {
            const int save = cfg.method;
            cfg.method = method;
            try {
                raise_state();
            } catch (...) {
                cfg.method = save;
                throw;
            }
        }
        return (uint64_t)hs->q_row;
    }
    void query(double theta, bool want_set) {
        not_sharded("greedy threshold / index-set queries");
        reset_status();
        launch_query(P, stream, theta, want_set ? 1 : 0);
        pull_state();
        if (hs->status == ST_ERROR) {
            launch_ctrl(st.p, k, k, FIN_ITERATION, 0, 1, stream);
            fail(AXB_DOMAIN_ERROR, "greedy threshold: zero residual");
        }
    }
};

// =========================================================================
// C-ABI
namespace {

// Entry points on a created handle run on the handle's device and restore the
// caller's current device afterwards, so handles on several devices can be
// driven from one host thread (streams, events and launches are per device).
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(const axb_solver* s) {
        if (!s || !s->stream) return;  // not created yet: create() selects the device
        int cur = 0;
        if (cudaGetDevice(&cur) == cudaSuccess && cur != s->opt.device &&
            cudaSetDevice(s->opt.device) == cudaSuccess)
            prev = cur;
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

template <class F>
int guarded(axb_solver* s, F&& f) {
    DeviceScope scope(s);
    try {
        f();
        return AXB_OK;
    } catch (const AxbError& e) {
        if (s) {
            s->err = e.msg;
            s->err_k = e.k;
            s->err_val = e.val;
        }
        return e.code;
    } catch (const std::exception& e) {
        if (s) s->err = e.what();
        return AXB_CUDA_ERROR;
    }
}
}  // namespace

extern "C" {

void axb_options_default(axb_options* o) {
    std::memset(o, 0, sizeof *o);
    o->cache_gram = -1;
    o->spectral_on_device = -1;
    o->tie_guard = 1;
    o->world_size = 1;
}

int axb_checked_build(void) {
#ifdef AXB_CHECKED
    return 1;
#else
    return 0;
#endif
}
int axb_abi_version(void) { return AXB_B200_ABI_VERSION; }

int axb_nccl_unique_id(unsigned char out[128]) {
    const char* why = "";
    const axb_nccl::Api* a = axb_nccl::api(&why);
    if (!a) {
        g_create_err = why;
        return AXB_CUDA_ERROR;
    }
    ncclUniqueId id;
    if (a->GetUniqueId(&id) != ncclSuccess) return AXB_CUDA_ERROR;
    std::memcpy(out, id.internal, 128);
    return AXB_OK;
}

int axb_nccl_comm_create(int nranks, const unsigned char id[128], int rank, int device,
                         void** comm) {
    const char* why = "";
    const axb_nccl::Api* a = axb_nccl::api(&why);
    if (!a) {
        g_create_err = why;
        return AXB_CUDA_ERROR;
    }
    if (cudaSetDevice(device) != cudaSuccess) return AXB_CUDA_ERROR;
    ncclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    ncclComm_t c = nullptr;
    const ncclResult_t r = a->CommInitRank(&c, nranks, uid, rank);
    if (r != ncclSuccess) {
        g_create_err = a->GetErrorString(r);
        return AXB_CUDA_ERROR;
    }
    *comm = c;
    return AXB_OK;
}

int axb_nccl_emulated_group(int world, void** comms) {
    if (world < 1 || !comms) return AXB_CONFIG_ERROR;
    axb_nccl::emulated_group(world, comms);
    return AXB_OK;
}
int axb_nccl_comm_destroy(void* comm) {
    if (comm && axb_nccl::is_emulated(comm))
        return axb_nccl::emulated_api()->CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess
                   ? AXB_OK : AXB_CUDA_ERROR;
    const axb_nccl::Api* a = axb_nccl::api(nullptr);
    if (!a || !comm) return AXB_OK;
    return a->CommDestroy(static_cast<ncclComm_t>(comm)) == ncclSuccess ? AXB_OK : AXB_CUDA_ERROR;
}

int axb_device_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return 0;
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, 0) != cudaSuccess) return 0;
    return p.major >= 10 ? 1 : 0;
}

const char* axb_last_create_error(void) { return g_create_err.c_str(); }

int axb_solver_create(const double* A, uint64_t m, uint64_t p, const double* B, uint64_t q,
                      uint64_t n, const double* C, const double* X0, const axb_config* cfg,
                      const axb_options* opt, axb_solver** out) {
    *out = nullptr;
    auto s = std::make_unique<axb_solver>();
    s->m = m; s->p = p; s->q = q; s->n = n;
    s->cfg = *cfg;
    if (opt) s->opt = *opt;
    else axb_options_default(&s->opt);
    int prev_dev = -1;
    if (cudaGetDevice(&prev_dev) != cudaSuccess) prev_dev = -1;
    cudaGetLastError();
    int st = guarded(s.get(), [&] { s->create(A, B, C, X0); });
    if (st != AXB_OK) {
        g_create_err = s->err;
        s.reset();  // released on its own device
    } else {
        g_create_err.clear();
        *out = s.release();
    }
    if (prev_dev >= 0) cudaSetDevice(prev_dev);  // the caller's current device is left as it was
    if (st != AXB_OK) return st;
    return AXB_OK;
}

namespace {
int expand(const axb_matrix* M, std::vector<double>& out, const char* name, bool fill = true);
int check_csr(const axb_matrix* M, const char* name) {
    std::vector<double> none;
    return expand(M, none, name, false);
}
// SparseMatrix::validate (matrix.hpp:94-175) + expansion to row-major dense
int expand(const axb_matrix* M, std::vector<double>& out, const char* name, bool fill) {
    if (M->kind == 0) return AXB_OK;
    if (M->kind != 1) {
        g_create_err = std::string(name) + ": unknown matrix kind";
        return AXB_CONFIG_ERROR;
    }
    const uint64_t r = M->rows, c = M->cols;
    if (!M->row_ptr || (M->nnz && (!M->col_idx || !M->values)) || M->row_ptr[0] != 0 ||
        M->row_ptr[r] != M->nnz) {
        g_create_err = std::string(name) + ": malformed CSR row pointer";
        return AXB_SHAPE_ERROR;
    }
    if (fill) out.assign(r * c, 0.0);
    for (uint64_t i = 0; i < r; ++i) {
        if (M->row_ptr[i + 1] < M->row_ptr[i]) {
            g_create_err = std::string(name) + ": CSR row pointer decreases";
            return AXB_SHAPE_ERROR;
        }
        for (uint64_t t = M->row_ptr[i]; t < M->row_ptr[i + 1]; ++t) {
            const uint64_t j = M->col_idx[t];
            const double v = M->values[t];
            if (j >= c || (t > M->row_ptr[i] && j <= M->col_idx[t - 1])) {
                g_create_err = std::string(name) + ": CSR column indices must ascend within a row";
                return AXB_SHAPE_ERROR;
            }
            if (!std::isfinite(v) || v == 0.0) {
                g_create_err = std::string(name) + ": CSR values must be finite and nonzero";
                return AXB_DOMAIN_ERROR;
            }
            if (fill) out[i * c + j] = v;
        }
    }
    return AXB_OK;
}
}  // namespace

extern "C++" {
namespace axb_dev {  // shared with axb_analysis.cu
std::string& handleless_error() { return g_create_err; }
int expand_matrix(const axb_matrix* M, std::vector<double>& out, const char* name) {
    return expand(M, out, name);
}
}  // namespace axb_dev
}

int axb_solver_create_ex(const axb_matrix* A, const axb_matrix* B, const double* C,
                         const double* X0, const axb_config* cfg, const axb_options* opt,
                         axb_solver** out) {
    *out = nullptr;
    if (opt && opt->inputs_on_device && (A->kind == 1 || B->kind == 1)) {
        g_create_err = "CSR operands are host arrays";
        return AXB_CONFIG_ERROR;
    }
    std::vector<double> Ad, Bd;
    int st = A->kind == 1 ? check_csr(A, "A") : expand(A, Ad, "A");
    if (st) return st;
    st = expand(B, Bd, "B");  // B's dense copy serves ‖B‖₂ and the residual GEMM
    if (st) return st;
    if (opt && opt->nccl_comm && A->kind == 1) {  // row sharding takes dense operands
        st = expand(A, Ad, "A");
        if (st) return st;
    }
    const bool sparse = (A->kind == 1 || B->kind == 1) && !(opt && opt->nccl_comm);
    *out = nullptr;
    auto s = std::make_unique<axb_solver>();
    s->m = A->rows; s->p = A->cols; s->q = B->rows; s->n = B->cols;
    s->cfg = *cfg;
    if (opt) s->opt = *opt;
    else axb_options_default(&s->opt);
    if (sparse) {
        s->in_A = A;
        s->in_B = B;
    }
    int prev_dev = -1;
    if (cudaGetDevice(&prev_dev) != cudaSuccess) prev_dev = -1;
    cudaGetLastError();
    const double* a_dense = A->kind == 1 ? (Ad.empty() ? nullptr : Ad.data()) : A->dense;
    const double* b_dense = B->kind == 1 ? Bd.data() : B->dense;
    st = guarded(s.get(), [&] { s->create(a_dense, b_dense, C, X0); });
    s->in_A = s->in_B = nullptr;  // borrowed for create() only
    if (st != AXB_OK) {
        g_create_err = s->err;
        s.reset();
    } else {
        g_create_err.clear();
        *out = s.release();
    }
    if (prev_dev >= 0) cudaSetDevice(prev_dev);
    return st;
}

void axb_solver_destroy(axb_solver* s) {
    DeviceScope scope(s);
    delete s;
}
const char* axb_solver_last_error(const axb_solver* s) { return s->err.c_str(); }

int axb_solver_step(axb_solver* s, uint64_t* row) {
    return guarded(s, [&] { s->steps(1, row, false); });
}
int axb_solver_steps(axb_solver* s, uint64_t k, uint64_t* rows, int32_t mirror_refresh) {
    return guarded(s, [&] { s->steps(k, rows, mirror_refresh != 0); });
}
int axb_solver_replay(axb_solver* s, uint64_t k, const uint64_t* rows, int32_t mirror_refresh) {
    return guarded(s, [&] { s->replay(k, rows, mirror_refresh != 0); });
}
int axb_solver_update_row(axb_solver* s, uint64_t i) {
    return guarded(s, [&] { s->update_row(i); });
}
int axb_solver_run(axb_solver* s, axb_report* rep, uint64_t* trace_k, double* trace_rrn,
                   double* trace_rel, uint64_t* trace_row, uint64_t trace_cap, double* x_out) {
    return guarded(s, [&] { s->run(rep, trace_k, trace_rrn, trace_rel, trace_row, trace_cap, x_out); });
}
namespace {
// per-device launch resources of axb_solvers_run
struct BatchRes {
    cudaStream_t s = nullptr;
    Params* dP = nullptr;
    Params* hP = nullptr;  // pinned staging
    size_t cap = 0;
};
std::mutex g_batch_mu;
BatchRes g_batch[64];

int record_failure(axb_solver* s, const AxbError& e) {
    s->err = e.msg;
    s->err_k = e.k;
    s->err_val = e.val;
    return e.code;
}
}  // namespace

int axb_solvers_run(axb_solver* const* hs, uint32_t count, axb_report* reps,
                    double* const* x_outs, int32_t* statuses) {
    if (count == 0) return AXB_OK;
    if (!hs || !reps || !statuses) {
        g_create_err = "axb_solvers_run: null argument";
        return AXB_CONFIG_ERROR;
    }
    for (uint32_t i = 0; i < count; ++i) {
        if (!hs[i]) {
            g_create_err = "axb_solvers_run: null handle";
            return AXB_CONFIG_ERROR;
        }
        if (hs[i]->opt.device != hs[0]->opt.device) {
            g_create_err = "axb_solvers_run: all handles must live on one device";
            return AXB_CONFIG_ERROR;
        }
        if (hs[i]->sharded) {
            g_create_err = "axb_solvers_run: sharded handles run on their own (axb_solver_run)";
            return AXB_CONFIG_ERROR;
        }
        for (uint32_t j = 0; j < i; ++j)
            if (hs[j] == hs[i]) {
                g_create_err = "axb_solvers_run: duplicate handle";
                return AXB_CONFIG_ERROR;
            }
    }
    const int dev = hs[0]->opt.device;
    std::lock_guard<std::mutex> lock(g_batch_mu);
    int prev = 0;
    cudaGetDevice(&prev);
    if (cudaSetDevice(dev) != cudaSuccess) {
        g_create_err = "axb_solvers_run: cudaSetDevice failed";
        return AXB_CUDA_ERROR;
    }
    BatchRes& br = g_batch[dev & 63];
    std::vector<axb_solver::RunCtx> ctx(count);
    std::vector<char> active(count, 0);
    for (uint32_t i = 0; i < count; ++i) {
        statuses[i] = AXB_OK;
        ctx[i].rep = &reps[i];
        ctx[i].x_out = x_outs ? x_outs[i] : nullptr;
        try {
            hs[i]->run_begin(ctx[i]);
            active[i] = 1;
        } catch (const AxbError& e) {
            statuses[i] = record_failure(hs[i], e);
        }
    }
    // Batched wall-clock semantics: every handle's loop clock starts at one common
    // instant, after all the run_begin() work (each handle's initial exact metric,
    // solver.hpp:344, which the reference also runs before its clock starts), and
    // ends when that handle's own loop ends.  Handles advance together through
    // shared launches, so a handle's wall time covers the batch's progress up to
    // its own end — it is the time-to-solution inside this batch, not the time the
    // handle would take alone (use axb_solver_run for that).
    {
        const auto common = std::chrono::steady_clock::now();
        for (uint32_t i = 0; i < count; ++i)
            if (active[i]) ctx[i].t0 = common;
    }
    auto fail_one = [&](uint32_t i, const AxbError& e) {
        hs[i]->run_fail(ctx[i], e);
        statuses[i] = record_failure(hs[i], e);
        active[i] = 0;
    };
    int rc = AXB_OK;
    try {
        for (;;) {
            std::vector<uint32_t> group;
            bool any = false;
            for (uint32_t i = 0; i < count; ++i) {
                if (!active[i]) continue;
                axb_solver* h = hs[i];
                try {
                    if (!h->run_segment(ctx[i])) {
                        h->run_end(ctx[i]);
                        active[i] = 0;
                        continue;
                    }
                    any = true;
                    if (h->batchable()) {
                        h->batch_launch(ctx[i].nb, 1, true);
                        group.push_back(i);
                    } else {  // large systems keep their own launch path
                        h->run_after(ctx[i], h->batch(ctx[i].nb, 1));
                    }
                } catch (const AxbError& e) {
                    fail_one(i, e);
                }
            }
            if (!any) break;
            if (group.empty()) continue;
            // every armed control block must land before the shared launch reads it
            for (uint32_t i : group) ck(cudaStreamSynchronize(hs[i]->stream), "arm");
            if (!br.s) ck(cudaStreamCreateWithFlags(&br.s, cudaStreamNonBlocking), "batch stream");
            if (br.cap < group.size()) {
                if (br.dP) cudaFree(br.dP);
                if (br.hP) cudaFreeHost(br.hP);
                br.dP = nullptr;
                br.hP = nullptr;
                br.cap = 0;
                const size_t want = std::max<size_t>(group.size(), 256);
                ck(cudaMalloc(&br.dP, sizeof(Params) * want), "batch params");
                ck(cudaMallocHost(&br.hP, sizeof(Params) * want), "batch params");
                br.cap = want;
            }
            long long max_m = 1;
            for (size_t j = 0; j < group.size(); ++j) {
                br.hP[j] = hs[group[j]]->P;
                max_m = std::max<long long>(max_m, hs[group[j]]->P.m);
            }
            ck(cudaMemcpyAsync(br.dP, br.hP, sizeof(Params) * group.size(), cudaMemcpyHostToDevice,
                               br.s), "batch params");
            const int e = launch_persist_batch(br.dP, (int)group.size(), max_m, br.s);
            if (e != 0) ck(static_cast<cudaError_t>(e), "batched persistent kernel launch");
            ck(cudaStreamSynchronize(br.s), "batched persistent kernel");
            for (uint32_t i : group) {
                try {
                    hs[i]->run_after(ctx[i], hs[i]->batch_collect());
                } catch (const AxbError& e) {
                    fail_one(i, e);
                }
            }
        }
    } catch (const AxbError& e) {  // launch-level failure: every open run fails
        g_create_err = e.msg;
        rc = e.code;
        for (uint32_t i = 0; i < count; ++i)
            if (active[i]) {
                hs[i]->run_fail(ctx[i], e);
                statuses[i] = record_failure(hs[i], e);
            }
    }
    cudaSetDevice(prev);
    return rc;
}

int axb_solver_select_cyclic(axb_solver* s, uint64_t* row) {
    return guarded(s, [&] { *row = s->select_consume(AXB_BK, 0.5); });
}
int axb_solver_select_rbk(axb_solver* s, uint64_t* row) {
    return guarded(s, [&] { *row = s->select_consume(AXB_RBK, 0.5); });
}
int axb_solver_select_greedy(axb_solver* s, double theta, uint64_t* row) {
    return guarded(s, [&] { *row = s->select_consume(AXB_GRBK, theta); });
}
int axb_solver_select_mwrbk(axb_solver* s, uint64_t* row) {
    return guarded(s, [&] { *row = s->select_consume(AXB_MWRBK, 0.5); });
}
int axb_solver_greedy_threshold(axb_solver* s, double theta, double* out) {
    return guarded(s, [&] {
        s->query(theta, false);
        *out = s->hs->q_zeta;
    });
}
int axb_solver_rgrbk_threshold(axb_solver* s, double theta, double* out) {
    return guarded(s, [&] {
        if (!(theta > 0.0 && theta < 1.0)) fail(AXB_CONFIG_ERROR, "theta must lie in (0, 1)");
        s->query(theta, false);
        *out = s->hs->q_zeta;
    });
}
int axb_solver_greedy_index_set(axb_solver* s, double theta, uint64_t* out, uint64_t* count) {
    return guarded(s, [&] {
        s->query(theta, true);
        std::vector<int> f(s->m);
        ck(cudaMemcpy(f.data(), s->flags.p, sizeof(int) * s->m, cudaMemcpyDeviceToHost), "flags");
        uint64_t c = 0;
        for (uint64_t i = 0; i < s->m; ++i)
            if (f[i]) out[c++] = i;
        if (c == 0) fail(AXB_INVARIANT_ERROR, "greedy index set is empty");
        *count = c;
    });
}
int axb_solver_max_residual_ratio(axb_solver* s, uint64_t* row, double* ratio) {
    return guarded(s, [&] {
        s->pull_state();
        if (s->hs->argmax < 0 || s->hs->argmax >= (long long)s->m)
            fail(AXB_DOMAIN_ERROR, "no nonzero row in A");
        *row = (uint64_t)s->hs->argmax;
        *ratio = s->hs->max_ratio;
    });
}
int axb_solver_current_metric(axb_solver* s, double* out) {
    return guarded(s, [&] { *out = s->current_metric(); });
}
int axb_solver_current_residual_rel(axb_solver* s, double* out) {
    return guarded(s, [&] { *out = s->current_residual_rel(); });
}
int axb_solver_exact_metric(axb_solver* s, double* out) {
    return guarded(s, [&] { *out = s->exact_metric(); });
}
int axb_solver_exact_residual_rel(axb_solver* s, double* out) {
    return guarded(s, [&] { *out = s->exact_residual_rel(); });
}
int axb_solver_residual_drift(axb_solver* s, double* out) {
    return guarded(s, [&] { *out = s->residual_drift(); });
}
int axb_solver_checkpoint(axb_solver* s) {
    return guarded(s, [&] { s->checkpoint(); });
}
uint64_t axb_solver_iteration(const axb_solver* s) { return s->k; }
double axb_solver_alpha(const axb_solver* s) { return s->alpha; }
double axb_solver_spectral_norm_b(const axb_solver* s) { return s->b_spec; }
int axb_solver_alpha_outside_bound(const axb_solver* s) { return s->alpha_outside ? 1 : 0; }
int axb_solver_gram_cached(const axb_solver* s) { return s->gram_cached ? 1 : 0; }
double axb_solver_a_fro_sq(const axb_solver* s) { return s->a_fro_sq; }
int axb_solver_residual_fro_sq(axb_solver* s, double* out) {
    return guarded(s, [&] {
        s->pull_state();
        *out = s->hs->r_fro_sq;
    });
}
static int copy_out(axb_solver* s, double* dst, const double* src, size_t count) {
    return guarded(s, [&] {
        d2h_copy(dst, src, sizeof(double) * count, s->stream);
    });
}
int axb_solver_get_X(axb_solver* s, double* out) {
    const int st = guarded(s, [&] {
        s->gather_X();
        s->sync("gather X");
    });
    return st ? st : copy_out(s, out, s->X.p, s->p * s->q);
}
int axb_solver_get_R(axb_solver* s, double* out) { return copy_out(s, out, s->R.p, s->m * s->n); }
int axb_solver_get_r_sq(axb_solver* s, double* out) {
    return copy_out(s, out, s->P.r_sq, s->m);  // sharded: this rank's slice of the global r_sq
}
int axb_solver_get_a_sq(axb_solver* s, double* out) { return copy_out(s, out, s->a_sq.p, s->m); }
int axb_solver_dims(const axb_solver* s, uint64_t dims[4]) {
    dims[0] = s->m; dims[1] = s->p; dims[2] = s->q; dims[3] = s->n;
    return AXB_OK;
}
int axb_solver_last_timing(const axb_solver* s, double* loop_ms, double* k2_ms,
                           uint64_t* k2_launches, uint64_t* kernel_launches) {
    if (loop_ms) *loop_ms = s->loop_ms;
    if (k2_ms) *k2_ms = s->k2_ms;
    if (k2_launches) *k2_launches = s->k2_launches;
    if (kernel_launches) *kernel_launches = s->kernel_launches;
    return AXB_OK;
}
int axb_solver_last_error_info(const axb_solver* s, uint64_t* iteration, double* value) {
    if (iteration) *iteration = s->err_k;
    if (value) *value = s->err_val;
    return AXB_OK;
}
int axb_solver_debug_state(axb_solver* s, uint64_t out[8]) {
    return guarded(s, [&] {
        s->pull_state();
        for (int i = 0; i < 8; ++i) out[i] = s->hs->dbg[i];
    });
}
int axb_debug_timeline(uint64_t out[512], int32_t reset) {
    return axb_dev::timeline_read(reinterpret_cast<unsigned long long*>(out), reset);
}
int axb_debug_dgemm(const double* A, const double* B, const double* Cin, double* D, uint64_t M,
                    uint64_t N, uint64_t K, int32_t b_trans, int32_t reps, double* ms) {
    if (!A || !B || !D || !ms || reps <= 0) return AXB_CONFIG_ERROR;
    axb_dev::GemmArgs g{};
    g.M = (long long)M;
    g.N = (long long)N;
    g.K = (long long)K;
    g.A = A;
    g.lda = (long long)K;
    g.B = B;
    g.ldb = (long long)(b_trans ? K : N);
    g.b_trans = b_trans;
    g.D = D;
    g.ldd = (long long)N;
    g.Cin = Cin;
    g.ldc = (long long)N;
    g.store = 1;
    cudaEvent_t e0, e1;
    if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
        return AXB_CUDA_ERROR;
    axb_dev::launch_gemm(g, 0);
    cudaEventRecord(e0, 0);
    for (int r = 0; r < reps; ++r) axb_dev::launch_gemm(g, 0);
    cudaEventRecord(e1, 0);
    const cudaError_t err = cudaEventSynchronize(e1);
    float t = 0.f;
    cudaEventElapsedTime(&t, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *ms = (double)t / reps;
    return err == cudaSuccess && cudaGetLastError() == cudaSuccess ? AXB_OK : AXB_CUDA_ERROR;
}
int axb_solver_kernel_times(const axb_solver* s, double out_ms[3]) {
    const double nl = s->k2_launches ? (double)s->k2_launches : 1.0;
    out_ms[0] = s->yg_ms / nl;
    out_ms[1] = s->zx_ms / nl;
    out_ms[2] = s->k2_ms / nl;
    return AXB_OK;
}
int axb_solver_collective_times(const axb_solver* s, double out_ms[5]) {
    const double nl = s->k2_launches ? (double)s->k2_launches : 1.0;
    out_ms[0] = s->coll_ms[0] / nl;
    out_ms[1] = s->coll_ms[1] / nl;
    out_ms[2] = s->coll_ms[2] / nl;
    out_ms[3] = s->sel_ms / nl;
    out_ms[4] = s->coll_ms[3] / nl;
    return AXB_OK;
}
int axb_solver_set_profiling(axb_solver* s, int32_t on) {
    s->profiling = on != 0;
    s->k2_ms = 0.0;
    s->yg_ms = 0.0;
    s->zx_ms = 0.0;
    s->sel_ms = 0.0;
    for (double& c : s->coll_ms) c = 0.0;
    s->k2_launches = 0;
    s->kernel_launches = 0;
    return AXB_OK;
}

}  // extern "C"
