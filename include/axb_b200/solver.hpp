// axb_b200/solver.hpp — header-only C++ drop-in over the C-ABI (axb_b200.h).
//
// Restores the shapes of the reference's engine API (solver.hpp:16-532):
// Method, AlphaRule, StopRule, SolveConfig, TracePoint, SolveReport, Solver and
// solve(), with errors rethrown as exceptions.  When the reference headers are
// on the include path (<axb/errors.hpp>), the reference's own exception types
// are thrown (axb::ShapeError, axb::DivergenceError{iteration,residual_norm},
// …), so existing catch sites keep working; otherwise an equivalent taxonomy
// is defined here.  Matrices: any type with rows(), cols() and contiguous
// row-major double storage via data() (axb::DenseMatrix qualifies,
// matrix.hpp:37-89), or raw pointers.
//
//   axb::SolveReport r = axb::solve(A, B, C, X0, cfg);        // reference
//   axb_b200::SolveReport r = axb_b200::solve(A, B, C, X0, cfg);  // B200
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../axb_b200.h"

#if defined(__has_include)
#if __has_include(<axb/errors.hpp>)
#include <axb/errors.hpp>
#define AXB_B200_REFERENCE_ERRORS 1
#endif
#if __has_include(<axb/solver.hpp>) && !defined(AXB_B200_NO_REFERENCE_TYPES)
#include <axb/solver.hpp>
#define AXB_B200_REFERENCE_TYPES 1
#endif
#endif

namespace axb_b200 {

#ifdef AXB_B200_REFERENCE_ERRORS
using Error = axb::Error;
using ShapeError = axb::ShapeError;
using DomainError = axb::DomainError;
using CapacityError = axb::CapacityError;
using ConfigError = axb::ConfigError;
using ConvergenceError = axb::ConvergenceError;
using DivergenceError = axb::DivergenceError;
using InvariantError = axb::InvariantError;
using DecompositionError = axb::DecompositionError;
#else
// errors.hpp:10-72, restated
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct CapacityError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct ConvergenceError : Error {
    ConvergenceError(const std::string& msg, double estimate) : Error(msg), last_estimate(estimate) {}
    double last_estimate;
};
struct DivergenceError : Error {
    DivergenceError(std::size_t k, double residual)
        : Error("divergence at iteration " + std::to_string(k) + ", residual frobenius norm " +
                std::to_string(residual)),
          iteration(k), residual_norm(residual) {}
    std::size_t iteration;
    double residual_norm;
};
struct InvariantError : Error { using Error::Error; };
struct DecompositionError : Error { using Error::Error; };
#endif
/// Device/runtime failure (no reference analogue): no sm_100 device, CUDA error.
struct CudaError : Error {
    using Error::Error;
};

[[noreturn]] inline void throw_status(int code, const std::string& msg, std::uint64_t k = 0,
                                      double val = 0.0) {
    switch (code) {
        case AXB_SHAPE_ERROR: throw ShapeError(msg);
        case AXB_DOMAIN_ERROR: throw DomainError(msg);
        case AXB_CONFIG_ERROR: throw ConfigError(msg);
        case AXB_DIVERGENCE_ERROR: throw DivergenceError(k, val);
        case AXB_INVARIANT_ERROR: throw InvariantError(msg);
        case AXB_CONVERGENCE_ERROR: throw ConvergenceError(msg, val);
        case AXB_CAPACITY_ERROR: throw CapacityError(msg);
        case AXB_DECOMPOSITION_ERROR: throw DecompositionError(msg);
        default: throw CudaError(msg);
    }
}

// ---- configuration (solver.hpp:16-138) ----
enum class MethodTag { BK = AXB_BK, RBK = AXB_RBK, GRBK = AXB_GRBK, RGRBK = AXB_RGRBK, MWRBK = AXB_MWRBK };

struct Method {
    MethodTag tag = MethodTag::RBK;
    std::optional<double> theta;
    static Method bk() { return {MethodTag::BK, {}}; }
    static Method rbk() { return {MethodTag::RBK, {}}; }
    static Method grbk() { return {MethodTag::GRBK, {}}; }
    static Method rgrbk(double t) { return {MethodTag::RGRBK, t}; }
    static Method mwrbk() { return {MethodTag::MWRBK, {}}; }
    void validate() const {
        if (tag == MethodTag::RGRBK) {
            if (!theta) throw ConfigError("rgrbk requires theta");
            if (!(*theta > 0.0 && *theta < 1.0)) throw ConfigError("theta must lie strictly in (0, 1)");
        } else if (theta) {
            throw ConfigError("theta is only valid for rgrbk");
        }
    }
    std::string label() const {
        switch (tag) {
            case MethodTag::BK: return "bk";
            case MethodTag::RBK: return "rbk";
            case MethodTag::GRBK: return "grbk";
            case MethodTag::RGRBK: return "rgrbk";
            case MethodTag::MWRBK: return "mwrbk";
        }
        return "?";
    }
};

enum class AlphaRule { Safe = AXB_ALPHA_SAFE, Paper = AXB_ALPHA_PAPER, Fixed = AXB_ALPHA_FIXED };

struct StopRule {
    enum class Kind { SolutionRrn = AXB_STOP_SOLUTION_RRN, ResidualRel = AXB_STOP_RESIDUAL_REL };
    Kind kind = Kind::ResidualRel;
    double tol = 1e-6;
    std::vector<double> reference;  // p×q row-major (SolutionRrn)
    static StopRule solution_rrn(double tol, std::vector<double> ref) {
        return {Kind::SolutionRrn, tol, std::move(ref)};
    }
    template <class M>
    static StopRule solution_rrn(double tol, const M& ref) {
        const double* d = ref.data().data();
        return {Kind::SolutionRrn, tol, std::vector<double>(d, d + ref.rows() * ref.cols())};
    }
    static StopRule residual_rel(double tol) { return {Kind::ResidualRel, tol, {}}; }
};

struct SolveConfig {
    Method method = Method::rbk();
    AlphaRule alpha_rule = AlphaRule::Safe;
    double alpha_value = 0.0;
    StopRule stop = StopRule::residual_rel(1e-6);
    std::size_t max_iter = 200000;
    std::uint64_t seed = 0;
    bool record_trace = false;
    std::size_t refresh_interval = 1000;
};

struct TracePoint {
    std::size_t k;
    double rrn;
    double residual_rel;
    std::size_t selected_row;
};

enum class Terminated { Tolerance = AXB_TERMINATED_TOLERANCE, MaxIter = AXB_TERMINATED_MAX_ITER };

struct SolveReport {
    std::size_t iterations = 0;
    double wall_seconds = 0.0;
    double final_rrn = 0.0;
    double final_residual_rel = 0.0;
    Terminated terminated_by = Terminated::MaxIter;
    std::vector<TracePoint> trace;
    std::vector<double> X;  // p×q row-major
    double alpha = 0.0;
    std::uint64_t seed = 0;
    std::string method_label;
    bool alpha_outside_bound = false;
    std::size_t skipped_zero_rows = 0;
};

inline bool trace_point_due(std::size_t k) { return k < 10000 || k % 10 == 0; }
inline constexpr double kDriftGuardScale = 1e-8;

struct Options : axb_options {
    Options() { axb_options_default(this); }
};

/// axb::Solver<DenseMatrix,DenseMatrix> on a B200 (solver.hpp:143-515).
class Solver {
public:
    Solver(const double* A, std::size_t m, std::size_t p, const double* B, std::size_t q,
           std::size_t n, const double* C, const double* X0, SolveConfig cfg,
           const Options& opt = Options())
        : cfg_(std::move(cfg)), m_(m), p_(p), q_(q), n_(n) {
        cfg_.method.validate();
        // solver.hpp:182-185, before any buffer is handed to the library
        if (cfg_.stop.kind == StopRule::Kind::SolutionRrn && !cfg_.stop.reference.empty() &&
            cfg_.stop.reference.size() != p_ * q_)
            throw ShapeError("reference solution shape mismatch");
        const axb_config c = flat(cfg_);
        axb_solver* h = nullptr;
        const int st = axb_solver_create(A, m, p, B, q, n, C, X0, &c, &opt, &h);
        if (st) throw_status(st, axb_last_create_error());
        h_.reset(h);
    }
    /// Dense operands (any type with rows(), cols() and row-major data(), e.g.
    /// axb::DenseMatrix).  Shapes are checked BEFORE any buffer is read, as the
    /// reference's constructor does (solver.hpp:150-154): an undersized C or X0
    /// throws ShapeError instead of being copied past its end.
    template <class M>
    Solver(const M& A, const M& B, const M& C, const M& X0, SolveConfig cfg,
           const Options& opt = Options())
        : Solver(checked(A, B, C, X0), A.data().data(), A.rows(), A.cols(), B.data().data(),
                 B.rows(), B.cols(), C.data().data(), X0.data().data(), std::move(cfg), opt) {}

    /// Storage-agnostic operands (the reference's axb::Matrix variant, matrix.hpp:178):
    /// dense or CSR descriptors (axb_matrix), C m×n and X0 p×q dense (X0 may be null).
    Solver(const axb_matrix& A, const axb_matrix& B, const double* C, const double* X0,
           SolveConfig cfg, const Options& opt = Options())
        : cfg_(std::move(cfg)), m_(A.rows), p_(A.cols), q_(B.rows), n_(B.cols) {
        cfg_.method.validate();
        if (cfg_.stop.kind == StopRule::Kind::SolutionRrn && !cfg_.stop.reference.empty() &&
            cfg_.stop.reference.size() != p_ * q_)
            throw ShapeError("reference solution shape mismatch");
        const axb_config c = flat(cfg_);
        axb_solver* h = nullptr;
        const int st = axb_solver_create_ex(&A, &B, C, X0, &c, &opt, &h);
        if (st) throw_status(st, axb_last_create_error());
        h_.reset(h);
    }

    std::size_t step() {
        std::uint64_t r = 0;
        check(axb_solver_step(h_.get(), &r));
        return r;
    }
    std::vector<std::size_t> steps(std::size_t k, bool mirror_refresh = false) {
        std::vector<std::uint64_t> rows(k);
        check(axb_solver_steps(h_.get(), k, rows.data(), mirror_refresh ? 1 : 0));
        return {rows.begin(), rows.end()};
    }
    void replay(const std::vector<std::uint64_t>& rows, bool mirror_refresh = false) {
        check(axb_solver_replay(h_.get(), rows.size(), rows.data(), mirror_refresh ? 1 : 0));
    }
    void update_row(std::size_t i) { check(axb_solver_update_row(h_.get(), i)); }

    SolveReport run() {
        const std::size_t mi = cfg_.max_iter;
        const std::size_t cap = !cfg_.record_trace ? 0 : (mi <= 10000 ? mi : 10000 + (mi - 10000) / 10 + 1);
        std::vector<std::uint64_t> tk(cap), tr(cap);
        std::vector<double> trr(cap), trl(cap);
        SolveReport rep;
        rep.X.resize(p_ * q_);
        axb_report r{};
        const int st = axb_solver_run(h_.get(), &r, tk.data(), trr.data(), trl.data(), tr.data(),
                                      cap, rep.X.data());
        if (st) throw_status(st, axb_solver_last_error(h_.get()), r.diverged_iteration,
                             r.diverged_residual);
        rep.iterations = r.iterations;
        rep.wall_seconds = r.wall_seconds;
        rep.final_rrn = r.final_rrn;
        rep.final_residual_rel = r.final_residual_rel;
        rep.terminated_by = static_cast<Terminated>(r.terminated_by);
        rep.alpha = r.alpha;
        rep.seed = r.seed;
        rep.method_label = cfg_.method.label();
        rep.alpha_outside_bound = r.alpha_outside_bound != 0;
        rep.skipped_zero_rows = r.skipped_zero_rows;
        const std::size_t nt = r.trace_len < cap ? r.trace_len : cap;
        for (std::size_t t = 0; t < nt; ++t) rep.trace.push_back({tk[t], trr[t], trl[t], tr[t]});
        return rep;
    }

    // selection rules (solver.hpp:197-258, 387-400)
    std::size_t select_cyclic() { return sel(axb_solver_select_cyclic); }
    std::size_t select_rbk() { return sel(axb_solver_select_rbk); }
    std::size_t select_greedy(double theta) {
        std::uint64_t r = 0;
        check(axb_solver_select_greedy(h_.get(), theta, &r));
        return r;
    }
    std::size_t select_grbk() { return select_greedy(0.5); }
    std::size_t select_mwrbk() { return sel(axb_solver_select_mwrbk); }
    double greedy_threshold(double theta) { return scalar_t(axb_solver_greedy_threshold, theta); }
    double grbk_threshold() { return greedy_threshold(0.5); }
    double rgrbk_threshold(double theta) { return scalar_t(axb_solver_rgrbk_threshold, theta); }
    std::vector<std::size_t> greedy_index_set(double theta) {
        std::vector<std::uint64_t> out(m_);
        std::uint64_t c = 0;
        check(axb_solver_greedy_index_set(h_.get(), theta, out.data(), &c));
        return {out.begin(), out.begin() + static_cast<std::ptrdiff_t>(c)};
    }
    std::pair<std::size_t, double> max_residual_ratio() {
        std::uint64_t r = 0;
        double v = 0.0;
        check(axb_solver_max_residual_ratio(h_.get(), &r, &v));
        return {r, v};
    }

    // metrics (solver.hpp:403-436)
    double current_metric() { return scalar(axb_solver_current_metric); }
    double current_residual_rel() { return scalar(axb_solver_current_residual_rel); }
    double exact_metric() { return scalar(axb_solver_exact_metric); }
    double exact_residual_rel() { return scalar(axb_solver_exact_residual_rel); }
    double residual_drift() { return scalar(axb_solver_residual_drift); }
    void checkpoint() { check(axb_solver_checkpoint(h_.get())); }

    // accessors (solver.hpp:376-385); copies from HBM
    std::size_t iteration() const { return axb_solver_iteration(h_.get()); }
    double alpha() const { return axb_solver_alpha(h_.get()); }
    double spectral_norm_b() const { return axb_solver_spectral_norm_b(h_.get()); }
    bool alpha_outside_bound() const { return axb_solver_alpha_outside_bound(h_.get()) != 0; }
    double a_fro_sq() const { return axb_solver_a_fro_sq(h_.get()); }
    double residual_fro_sq() { return scalar(axb_solver_residual_fro_sq); }
    std::vector<double> X() { return vec(axb_solver_get_X, p_ * q_); }
    std::vector<double> R() { return vec(axb_solver_get_R, m_ * n_); }
    std::vector<double> residual_row_sq() { return vec(axb_solver_get_r_sq, m_); }
    std::vector<double> a_row_sq() { return vec(axb_solver_get_a_sq, m_); }

private:
    struct Checked {};
    template <class M>
    static Checked checked(const M& A, const M& B, const M& C, const M& X0) {
        const std::size_t m = A.rows(), p = A.cols(), q = B.rows(), n = B.cols();
        if (X0.rows() != p || X0.cols() != q)
            throw ShapeError("solve: X0 must be " + std::to_string(p) + "x" + std::to_string(q));
        if (C.rows() != m || C.cols() != n)
            throw ShapeError("solve: C must be " + std::to_string(m) + "x" + std::to_string(n));
        return {};
    }
    Solver(Checked, const double* A, std::size_t m, std::size_t p, const double* B, std::size_t q,
           std::size_t n, const double* C, const double* X0, SolveConfig cfg, const Options& opt)
        : Solver(A, m, p, B, q, n, C, X0, std::move(cfg), opt) {}
    static axb_config flat(const SolveConfig& k) {
        axb_config c{};
        c.method = static_cast<int32_t>(k.method.tag);
        c.has_theta = k.method.theta ? 1 : 0;
        c.theta = k.method.theta.value_or(0.0);
        c.alpha_rule = static_cast<int32_t>(k.alpha_rule);
        c.stop_kind = static_cast<int32_t>(k.stop.kind);
        c.alpha_value = k.alpha_value;
        c.tol = k.stop.tol;
        c.reference = k.stop.reference.empty() ? nullptr : k.stop.reference.data();
        c.max_iter = k.max_iter;
        c.seed = k.seed;
        c.record_trace = k.record_trace ? 1 : 0;
        c.refresh_interval = k.refresh_interval;
        return c;
    }
    struct Del {
        void operator()(axb_solver* s) const { axb_solver_destroy(s); }
    };
    void check(int st) {
        if (!st) return;
        std::uint64_t k = 0;
        double v = 0.0;
        axb_solver_last_error_info(h_.get(), &k, &v);
        throw_status(st, axb_solver_last_error(h_.get()), k, v);
    }
    std::size_t sel(int (*fn)(axb_solver*, std::uint64_t*)) {
        std::uint64_t r = 0;
        check(fn(h_.get(), &r));
        return r;
    }
    double scalar(int (*fn)(axb_solver*, double*)) {
        double v = 0.0;
        check(fn(h_.get(), &v));
        return v;
    }
    double scalar_t(int (*fn)(axb_solver*, double, double*), double t) {
        double v = 0.0;
        check(fn(h_.get(), t, &v));
        return v;
    }
    std::vector<double> vec(int (*fn)(axb_solver*, double*), std::size_t len) {
        std::vector<double> out(len);
        check(fn(h_.get(), out.data()));
        return out;
    }

    SolveConfig cfg_;
    std::size_t m_, p_, q_, n_;
    std::unique_ptr<axb_solver, Del> h_;
};

/// axb::solve (solver.hpp:518-532).
template <class M>
SolveReport solve(const M& A, const M& B, const M& C, const M& X0, const SolveConfig& cfg,
                  const Options& opt = Options()) {
    return Solver(A, B, C, X0, cfg, opt).run();
}

#ifdef AXB_B200_REFERENCE_TYPES
// ---- the reference's own types in and out (reference headers on the include path) ----
// A call site switches from   axb::solve(A, B, C, X0, cfg)
//                        to   axb_b200::solve(A, B, C, X0, cfg)
// with the same argument types (axb::Matrix or axb::DenseMatrix operands,
// axb::SolveConfig) and the same result type (axb::SolveReport).

/// axb::SolveConfig (solver.hpp:100-109) → axb_b200::SolveConfig.
inline SolveConfig to_b200(const axb::SolveConfig& c) {
    SolveConfig o;
    o.method.tag = static_cast<MethodTag>(static_cast<int>(c.method.tag));
    o.method.theta = c.method.theta;
    o.alpha_rule = static_cast<AlphaRule>(static_cast<int>(c.alpha_rule));
    o.alpha_value = c.alpha_value;
    o.stop.kind = c.stop.kind == axb::StopRule::Kind::SolutionRrn ? StopRule::Kind::SolutionRrn
                                                                  : StopRule::Kind::ResidualRel;
    o.stop.tol = c.stop.tol;
    if (c.stop.reference) {
        if (o.stop.kind == StopRule::Kind::SolutionRrn &&
            (c.stop.reference->rows() == 0 || c.stop.reference->cols() == 0))
            throw ConfigError("solution_rrn stopping needs a reference solution");
        const auto d = c.stop.reference->data();
        o.stop.reference.assign(d.begin(), d.end());
    }
    o.max_iter = c.max_iter;
    o.seed = c.seed;
    o.record_trace = c.record_trace;
    o.refresh_interval = c.refresh_interval;
    return o;
}

/// axb_b200::SolveReport → axb::SolveReport (solver.hpp:120-133); X is p×q.
inline axb::SolveReport to_axb(SolveReport&& r, std::size_t p, std::size_t q) {
    axb::SolveReport o;
    o.iterations = r.iterations;
    o.wall_seconds = r.wall_seconds;
    o.final_rrn = r.final_rrn;
    o.final_residual_rel = r.final_residual_rel;
    o.terminated_by = r.terminated_by == Terminated::Tolerance ? axb::Terminated::Tolerance
                                                               : axb::Terminated::MaxIter;
    o.trace.reserve(r.trace.size());
    for (const auto& t : r.trace) o.trace.push_back({t.k, t.rrn, t.residual_rel, t.selected_row});
    o.X = axb::DenseMatrix(p, q, std::move(r.X));
    o.alpha = r.alpha;
    o.seed = r.seed;
    o.method_label = std::move(r.method_label);
    o.alpha_outside_bound = r.alpha_outside_bound;
    o.skipped_zero_rows = r.skipped_zero_rows;
    return o;
}

/// axb::Matrix (matrix.hpp:178: DenseMatrix or CSR SparseMatrix) → a borrowed
/// axb_matrix descriptor (valid while m lives).
inline axb_matrix describe(const axb::Matrix& m) {
    axb_matrix d{};
    if (const auto* dm = std::get_if<axb::DenseMatrix>(&m)) {
        d.kind = 0;
        d.rows = dm->rows();
        d.cols = dm->cols();
        d.dense = dm->data().data();
    } else {
        const auto& sm = std::get<axb::SparseMatrix>(m);
        d.kind = 1;
        d.rows = sm.rows();
        d.cols = sm.cols();
        d.nnz = sm.nnz();
        static_assert(sizeof(std::size_t) == sizeof(std::uint64_t), "CSR index width");
        d.row_ptr = reinterpret_cast<const std::uint64_t*>(sm.row_ptr().data());
        d.col_idx = sm.rows() ? reinterpret_cast<const std::uint64_t*>(sm.row_indices(0).data())
                              : nullptr;
        d.values = sm.rows() ? sm.row_values(0).data() : nullptr;
    }
    return d;
}

/// Drop-in for axb::solve(const Matrix&, const Matrix&, const DenseMatrix&,
/// const DenseMatrix&, const SolveConfig&) (solver.hpp:518-526): same arguments,
/// same axb::SolveReport, the reference's exception types.
inline axb::SolveReport solve(const axb::Matrix& A, const axb::Matrix& B, const axb::DenseMatrix& C,
                              const axb::DenseMatrix& X0, const axb::SolveConfig& cfg,
                              const Options& opt = Options()) {
    const axb_matrix a = describe(A), b = describe(B);
    if (X0.rows() != a.cols || X0.cols() != b.rows)
        throw ShapeError("solve: X0 must be " + std::to_string(a.cols) + "x" + std::to_string(b.rows));
    if (C.rows() != a.rows || C.cols() != b.cols)
        throw ShapeError("solve: C must be " + std::to_string(a.rows) + "x" + std::to_string(b.cols));
    Solver s(a, b, C.data().data(), X0.data().data(), to_b200(cfg), opt);
    return to_axb(s.run(), a.cols, b.rows);
}

/// Dense overload (solver.hpp:528-532).
inline axb::SolveReport solve(const axb::DenseMatrix& A, const axb::DenseMatrix& B,
                              const axb::DenseMatrix& C, const axb::DenseMatrix& X0,
                              const axb::SolveConfig& cfg, const Options& opt = Options()) {
    Solver s(A, B, C, X0, to_b200(cfg), opt);
    return to_axb(s.run(), A.cols(), B.rows());
}
#endif  // AXB_B200_REFERENCE_TYPES

}  // namespace axb_b200
