// Drop-in example: the reference's call pattern (axb::solve / Solver::step, as at
// axbsolve.cpp:200 and acceptance.cpp:128-141) compiled against the B200 shim.
// Prints "iterations=<k> rrn=<final> rows=<r0>,<r1>,<r2>" or "error=<type>: <msg>".
#include <cmath>
#include <cstdio>
#include <vector>

#include "axb_b200/solver.hpp"

struct Dense {  // minimal row-major stand-in for axb::DenseMatrix (matrix.hpp:37-89)
    std::size_t r, c;
    std::vector<double> v;
    std::size_t rows() const { return r; }
    std::size_t cols() const { return c; }
    const std::vector<double>& data() const { return v; }
};

int main() {
    const std::size_t m = 40, p = 10, q = 8, n = 30;
    Dense A{m, p, {}}, B{q, n, {}}, X{p, q, {}}, X0{p, q, std::vector<double>(p * q, 0.0)};
    for (std::size_t i = 0; i < m * p; ++i) A.v.push_back(std::sin(1.0 + 0.37 * i));
    for (std::size_t i = 0; i < q * n; ++i) B.v.push_back(std::cos(0.5 + 0.11 * i));
    for (std::size_t i = 0; i < p * q; ++i) X.v.push_back(std::sin(0.3 * i) + 0.5);
    Dense T{m, q, std::vector<double>(m * q, 0.0)}, C{m, n, std::vector<double>(m * n, 0.0)};
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t k = 0; k < p; ++k)
            for (std::size_t j = 0; j < q; ++j) T.v[i * q + j] += A.v[i * p + k] * X.v[k * q + j];
    for (std::size_t i = 0; i < m; ++i)
        for (std::size_t k = 0; k < q; ++k)
            for (std::size_t j = 0; j < n; ++j) C.v[i * n + j] += T.v[i * q + k] * B.v[k * n + j];
    axb_b200::SolveConfig cfg;
    cfg.method = axb_b200::Method::grbk();
    cfg.stop = axb_b200::StopRule::solution_rrn(1e-20, X.v);
    cfg.max_iter = 20000;
    cfg.seed = 42;
    try {
        axb_b200::Solver s(A, B, C, X0, cfg);
        const std::size_t r0 = s.step(), r1 = s.step(), r2 = s.step();
        axb_b200::SolveReport rep = s.run();
        std::printf("iterations=%zu rrn=%.3e rows=%zu,%zu,%zu\n", rep.iterations, rep.final_rrn, r0,
                    r1, r2);
    } catch (const axb_b200::CudaError& e) {
        std::printf("error=CudaError: %s\n", e.what());
        return 3;
    } catch (const axb_b200::Error& e) {
        std::printf("error=Error: %s\n", e.what());
        return 2;
    }
    return 0;
}
