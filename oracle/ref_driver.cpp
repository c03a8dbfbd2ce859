// ref_driver.cpp — builds the UNMODIFIED reference engine into oracle/_ref/libaxbref.so.
//
// Test infrastructure only.  This file contains no reference source: it #includes
// the reference headers where they lie (/root/reference/proj/include, passed with
// -I by oracle/Makefile) and exposes a flat extern "C" surface so pytest can drive
// `axb::Solver` (solver.hpp:143-515) through ctypes.  It pins the C restatement in
// oracle/axb_oracle.c and generates the golden vectors in tests/golden/.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "axb/analysis.hpp"
#include "axb/decomp.hpp"
#include "axb/imaging.hpp"
#include "axb/rng.hpp"
#include "axb/solver.hpp"

using namespace axb;

namespace {

struct RefConfig {  // same layout as orc_config / axb_config
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
};

struct RefReport {
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
    uint64_t diverged_iteration;
    double diverged_residual;
};

using DSolver = Solver<DenseMatrix, DenseMatrix>;

struct Handle {
    std::unique_ptr<DSolver> s;
    std::string err;
    uint64_t div_k = 0;
    double div_res = 0.0;
};

DenseMatrix mk(const double* p, size_t r, size_t c) {
    if (!p) return DenseMatrix(r, c);
    return DenseMatrix(r, c, std::vector<double>(p, p + r * c));
}

SolveConfig to_cfg(const RefConfig* c, size_t p, size_t q) {
    SolveConfig cfg;
    cfg.method.tag = static_cast<MethodTag>(c->method);
    if (c->has_theta) cfg.method.theta = c->theta;
    cfg.alpha_rule = static_cast<AlphaRule>(c->alpha_rule);
    cfg.alpha_value = c->alpha_value;
    if (c->stop_kind == 0)
        cfg.stop = StopRule::solution_rrn(c->tol, c->reference ? mk(c->reference, p, q)
                                                               : DenseMatrix());
    else
        cfg.stop = StopRule::residual_rel(c->tol);
    if (c->stop_kind == 0 && !c->reference) cfg.stop.reference.reset();
    cfg.max_iter = c->max_iter;
    cfg.seed = c->seed;
    cfg.record_trace = c->record_trace != 0;
    cfg.refresh_interval = c->refresh_interval;
    return cfg;
}

template <class F>
int guarded(Handle* h, F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) {
        h->err = e.what();
        return 1;
    } catch (const DomainError& e) {
        h->err = e.what();
        return 2;
    } catch (const ConfigError& e) {
        h->err = e.what();
        return 3;
    } catch (const DivergenceError& e) {
        h->err = e.what();
        h->div_k = e.iteration;
        h->div_res = e.residual_norm;
        return 4;
    } catch (const InvariantError& e) {
        h->err = e.what();
        return 5;
    } catch (const ConvergenceError& e) {
        h->err = e.what();
        return 6;
    } catch (const DecompositionError& e) {
        h->err = e.what();
        return 9;
    } catch (const std::exception& e) {
        h->err = e.what();
        return 99;
    }
}

}  // namespace

extern "C" {

// problems.hpp:345-364 generate() for Gaussian A and B, mirrored with the
// reference's own RngStream / dense_gaussian / matmul (problems.hpp itself needs
// nlohmann json, which the reference does not vendor).
void ref_generate_gaussian(uint64_t seed, size_t m, size_t p, size_t q, size_t n, double* A,
                           double* B, double* X, double* C) {
    RngStream root(seed);
    RngStream sa = root.substream(1), sb = root.substream(2), sx = root.substream(3);
    DenseMatrix a = dense_gaussian(sa, m, p);
    DenseMatrix b = dense_gaussian(sb, q, n);
    DenseMatrix x = dense_gaussian(sx, p, q);
    DenseMatrix c = matmul(matmul(a, x), b);
    if (A) std::memcpy(A, a.data().data(), sizeof(double) * m * p);
    if (B) std::memcpy(B, b.data().data(), sizeof(double) * q * n);
    if (X) std::memcpy(X, x.data().data(), sizeof(double) * p * q);
    if (C) std::memcpy(C, c.data().data(), sizeof(double) * m * n);
}

uint64_t ref_rng_stream(uint64_t seed, uint64_t count, uint64_t* out_u64, double* out_gauss) {
    RngStream r(seed), g(seed);
    for (uint64_t i = 0; i < count; ++i) {
        if (out_u64) out_u64[i] = r.next_u64();
        if (out_gauss) out_gauss[i] = g.gauss();
    }
    return count;
}

uint64_t ref_substream_seed(uint64_t seed, uint64_t t) { return RngStream(seed).substream(t).seed(); }

double ref_spectral_norm(const double* b, size_t rows, size_t cols, double tol, uint64_t max_iter,
                         int* status) {
    Handle h;
    double out = 0.0;
    *status = guarded(&h, [&] { out = spectral_norm(mk(b, rows, cols), tol, max_iter); });
    return out;
}

void* ref_solver_create(const double* A, size_t m, size_t p, const double* B, size_t q, size_t n,
                        const double* C, const double* X0, const RefConfig* cfg, int* status) {
    auto* h = new Handle();
    *status = guarded(h, [&] {
        h->s = std::make_unique<DSolver>(mk(A, m, p), mk(B, q, n), mk(C, m, n), mk(X0, p, q),
                                         to_cfg(cfg, p, q));
    });
    if (*status) {
        delete h;
        return nullptr;
    }
    return h;
}

void ref_solver_destroy(void* hp) { delete static_cast<Handle*>(hp); }

int ref_solver_step(void* hp, uint64_t* row) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { *row = h->s->step(); });
}

// Drives step() k times the way acceptance.cpp:128-141 does, mirroring run()'s
// refresh schedule (solver.hpp:359-360) when `mirror_refresh` is set.
int ref_solver_steps(void* hp, uint64_t k, uint64_t* rows, int mirror_refresh,
                     uint64_t refresh_interval) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] {
        for (uint64_t t = 0; t < k; ++t) {
            rows[t] = h->s->step();
            if (mirror_refresh && refresh_interval > 0 && h->s->iteration() % refresh_interval == 0)
                h->s->checkpoint();
        }
    });
}

int ref_solver_update_row(void* hp, uint64_t i) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { h->s->update_row(i); });
}

int ref_solver_greedy_threshold(void* hp, double theta, double* out) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { *out = h->s->greedy_threshold(theta); });
}

int ref_solver_greedy_index_set(void* hp, double theta, uint64_t* out, uint64_t* count) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] {
        auto v = h->s->greedy_index_set(theta);
        for (size_t k = 0; k < v.size(); ++k) out[k] = v[k];
        *count = v.size();
    });
}

int ref_solver_max_residual_ratio(void* hp, uint64_t* row, double* ratio) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] {
        auto pr = h->s->max_residual_ratio();
        *row = pr.first;
        *ratio = pr.second;
    });
}

int ref_solver_run(void* hp, RefReport* rep, uint64_t* trace_row, double* trace_rrn,
                   uint64_t trace_cap, double* x_out) {
    auto* h = static_cast<Handle*>(hp);
    std::memset(rep, 0, sizeof *rep);
    int st = guarded(h, [&] {
        SolveReport r = h->s->run();
        rep->iterations = r.iterations;
        rep->wall_seconds = r.wall_seconds;
        rep->final_rrn = r.final_rrn;
        rep->final_residual_rel = r.final_residual_rel;
        rep->terminated_by = r.terminated_by == Terminated::Tolerance ? 0 : 1;
        rep->alpha_outside_bound = r.alpha_outside_bound;
        rep->alpha = r.alpha;
        rep->seed = r.seed;
        rep->skipped_zero_rows = r.skipped_zero_rows;
        rep->trace_len = r.trace.size();
        for (size_t t = 0; t < r.trace.size() && t < trace_cap; ++t) {
            if (trace_row) trace_row[t] = r.trace[t].selected_row;
            if (trace_rrn) trace_rrn[t] = r.trace[t].rrn;
        }
        if (x_out) std::memcpy(x_out, r.X.data().data(), sizeof(double) * r.X.size());
    });
    rep->diverged_iteration = h->div_k;
    rep->diverged_residual = h->div_res;
    return st;
}

int ref_solver_checkpoint(void* hp) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { h->s->checkpoint(); });
}

double ref_solver_alpha(void* hp) { return static_cast<Handle*>(hp)->s->alpha(); }
double ref_solver_spectral_norm_b(void* hp) { return static_cast<Handle*>(hp)->s->spectral_norm_b(); }
double ref_solver_residual_fro_sq(void* hp) { return static_cast<Handle*>(hp)->s->residual_fro_sq(); }
double ref_solver_a_fro_sq(void* hp) { return static_cast<Handle*>(hp)->s->a_fro_sq(); }
uint64_t ref_solver_iteration(void* hp) { return static_cast<Handle*>(hp)->s->iteration(); }
double ref_solver_current_metric(void* hp) { return static_cast<Handle*>(hp)->s->current_metric(); }

int ref_solver_exact_metric(void* hp, double* out) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { *out = h->s->exact_metric(); });
}

int ref_solver_residual_drift(void* hp, double* out) {
    auto* h = static_cast<Handle*>(hp);
    return guarded(h, [&] { *out = h->s->residual_drift(); });
}

void ref_solver_get_X(void* hp, double* out) {
    auto& x = static_cast<Handle*>(hp)->s->X();
    std::memcpy(out, x.data().data(), sizeof(double) * x.size());
}
void ref_solver_get_R(void* hp, double* out) {
    auto& r = static_cast<Handle*>(hp)->s->R();
    std::memcpy(out, r.data().data(), sizeof(double) * r.size());
}
void ref_solver_get_r_sq(void* hp, double* out) {
    auto v = static_cast<Handle*>(hp)->s->residual_row_sq();
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}
void ref_solver_get_a_sq(void* hp, double* out) {
    auto v = static_cast<Handle*>(hp)->s->a_row_sq();
    std::memcpy(out, v.data(), sizeof(double) * v.size());
}
const char* ref_solver_last_error(void* hp) { return static_cast<Handle*>(hp)->err.c_str(); }

// ---- analysis.hpp / decomp.hpp: svd, pseudoinverse,
// reference_solution, bk_limit, rrn on dense operands; errors in ref_analysis_error().
static thread_local Handle g_an;

const char* ref_analysis_error() { return g_an.err.c_str(); }

int ref_svd(const double* M, size_t rows, size_t cols, size_t max_sweeps, double* U,
            double* sigma, double* V, size_t* rank) {
    return guarded(&g_an, [&] {
        SvdFactors f = svd(mk(M, rows, cols), max_sweeps);
        if (U) std::memcpy(U, f.U.data().data(), sizeof(double) * f.U.size());
        if (V) std::memcpy(V, f.V.data().data(), sizeof(double) * f.V.size());
        if (sigma)
            std::memcpy(sigma, f.singular_values.data(),
                        sizeof(double) * f.singular_values.size());
        if (rank) *rank = f.numeric_rank;
    });
}

int ref_pseudoinverse(const double* M, size_t rows, size_t cols, double rank_tol, double* P) {
    return guarded(&g_an, [&] {
        DenseMatrix p = pseudoinverse(mk(M, rows, cols), rank_tol);
        std::memcpy(P, p.data().data(), sizeof(double) * p.size());
    });
}

int ref_reference_solution(const double* A, size_t m, size_t p, const double* B, size_t q,
                           size_t n, const double* C, double rank_tol, double* X, int* kind,
                           double* residual_check) {
    return guarded(&g_an, [&] {
        Matrix a = mk(A, m, p), b = mk(B, q, n);
        ReferenceSolution r = reference_solution(a, b, mk(C, m, n), rank_tol);
        std::memcpy(X, r.X_star.data().data(), sizeof(double) * r.X_star.size());
        if (kind) *kind = static_cast<int>(r.kind);
        if (residual_check) *residual_check = r.residual_check;
    });
}

int ref_bk_limit(const double* A, size_t m, size_t p, const double* B, size_t q, size_t n,
                 const double* C, const double* X0, double* out) {
    return guarded(&g_an, [&] {
        Matrix a = mk(A, m, p), b = mk(B, q, n);
        DenseMatrix l = bk_limit(a, b, mk(C, m, n), mk(X0, p, q));
        std::memcpy(out, l.data().data(), sizeof(double) * l.size());
    });
}

int ref_rrn(const double* xk, const double* ref, size_t rows, size_t cols, double* out) {
    return guarded(&g_an, [&] { *out = rrn(mk(xk, rows, cols), mk(ref, rows, cols)); });
}

// ---- CSR operands and the §6 restoration shape -------------
// imaging.hpp:93-136 build_blur_operator(gaussian_kernel(ksize, sigma)) for an
// h×w image: returns nnz; fills rp (h·w+1), ci, v when non-NULL.
uint64_t ref_blur_operator(size_t h, size_t w, size_t ksize, double sigma, uint64_t* rp,
                           uint64_t* ci, double* v) {
    const SparseMatrix A = build_blur_operator(h, w, gaussian_kernel(ksize, sigma));
    if (rp) {
        auto r = A.row_ptr();
        for (size_t i = 0; i < r.size(); ++i) rp[i] = r[i];
        for (size_t i = 0; i < A.rows(); ++i) {
            auto idx = A.row_indices(i);
            auto val = A.row_values(i);
            for (size_t k = 0; k < idx.size(); ++k) {
                ci[r[i] + k] = idx[k];
                v[r[i] + k] = val[k];
            }
        }
    }
    return A.nnz();
}

// imaging.hpp:276-310 synthetic_test_image, column-stacked (stack_channels,
// :42-51): X (h·w)×3 row-major; and the paper's cross-channel matrix A_c (:139-141)
void ref_synthetic_stack(size_t h, size_t w, double* X, double* A_c) {
    const ChannelStack s = stack_channels(synthetic_test_image(h, w));
    const auto d = s.X.data();
    std::copy(d.begin(), d.end(), X);
    const DenseMatrix c = cross_channel_paper();
    std::copy(c.data().begin(), c.data().end(), A_c);
}

// The reference's sparse engine: Solver<SparseMatrix, BMat> (BMat CSR when b_rp is
// non-NULL, else dense), k step() calls; rows, X (p×q), r_sq (m), α out.
int ref_sparse_steps(const uint64_t* a_rp, const uint64_t* a_ci, const double* a_v, size_t m,
                     size_t p, const uint64_t* b_rp, const uint64_t* b_ci, const double* b_v,
                     const double* b_dense, size_t q, size_t n, const double* C, const double* X0,
                     const RefConfig* cfg, uint64_t k, uint64_t* rows, double* X_out,
                     double* r_sq_out, double* alpha_out, char* err) {
    Handle h;
    auto csr = [](const uint64_t* rp, const uint64_t* ci, const double* v, size_t r, size_t c) {
        std::vector<size_t> R(rp, rp + r + 1), I(ci, ci + rp[r]);
        std::vector<double> V(v, v + rp[r]);
        return SparseMatrix(r, c, std::move(R), std::move(I), std::move(V));
    };
    auto drive = [&](auto& s) {
        for (uint64_t t = 0; t < k; ++t) rows[t] = s.step();
        const auto x = s.X().data();
        std::copy(x.begin(), x.end(), X_out);
        const auto rs = s.residual_row_sq();
        std::copy(rs.begin(), rs.end(), r_sq_out);
        *alpha_out = s.alpha();
    };
    const int st = guarded(&h, [&] {
        SparseMatrix A = csr(a_rp, a_ci, a_v, m, p);
        if (b_rp) {
            Solver<SparseMatrix, SparseMatrix> s(std::move(A), csr(b_rp, b_ci, b_v, q, n),
                                                 mk(C, m, n), mk(X0, p, q), to_cfg(cfg, p, q));
            drive(s);
        } else {
            Solver<SparseMatrix, DenseMatrix> s(std::move(A), mk(b_dense, q, n), mk(C, m, n),
                                                mk(X0, p, q), to_cfg(cfg, p, q));
            drive(s);
        }
    });
    if (st && err) std::snprintf(err, 256, "%s", h.err.c_str());
    return st;
}

}  // extern "C"
