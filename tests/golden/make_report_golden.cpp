// Golden report / trace files from the REFERENCE's own writers (report.hpp:55-136,
// axbsolve.cpp:205-212) — test infrastructure for SURVEY §8 F4.
//
// Compiled against the unmodified reference headers and an nlohmann/json 3.11.3
// stand-in for the reference's vendored json.hpp (see make_report_golden.sh).
// Writes into tests/golden/report/:
//   trace.csv, report.json     an `axbsolve solve`-style config-1 run (ME-GRBK,
//                              A 500×100, B 80×400 from generate(), solution_rrn
//                              1e-12, trace on): trace_to_csv and
//                              solve_report_to_json + {"stop","tol"} dumped with dump(2)
//   run_raw.txt                the same SolveReport fields and every TracePoint as
//                              hex floats, so a restatement can be fed identical values
//   bench.csv, bench.json      benchmark_to_csv / benchmark_to_json of fixed rows
//                              (optional theta / speed-up, a field needing RFC-4180 quoting)
//   restore.csv                restore_metrics_to_csv of fixed rows
#include <cstdio>
#include <string>

#include "axb/analysis.hpp"
#include "axb/rng.hpp"
#include "axb/report.hpp"
#include "axb/solver.hpp"

using namespace axb;

int main(int argc, char** argv) {
    const std::string dir = argc > 1 ? argv[1] : "tests/golden/report";
    // generate() for two Gaussian sources (problems.hpp:345-364): substreams 1/2/3
    RngStream root(7);
    RngStream sa = root.substream(1), sb = root.substream(2), sx = root.substream(3);
    DenseMatrix A = dense_gaussian(sa, 500, 100), B = dense_gaussian(sb, 80, 400);
    DenseMatrix Xs = dense_gaussian(sx, 100, 80);
    DenseMatrix C = matmul(matmul(A, Xs), B);
    SolveConfig cfg;
    cfg.method = Method::grbk();
    cfg.stop = StopRule::solution_rrn(1e-12, Xs);
    cfg.max_iter = 1000000;
    cfg.seed = 42;
    cfg.record_trace = true;
    SolveReport rep = solve(A, B, C, DenseMatrix(100, 80), cfg);
    rep.wall_seconds = 1.25;  // fixed: wall time is not replayable (cli_tests.cpp:168-195)
    nlohmann::json rj = solve_report_to_json(rep);
    rj["stop"] = "rrn";
    rj["tol"] = 1e-12;
    write_text_file(dir + "/report.json", rj.dump(2) + "\n");
    write_text_file(dir + "/trace.csv", trace_to_csv(rep.trace));
    {
        FILE* f = std::fopen((dir + "/run_raw.txt").c_str(), "w");
        std::fprintf(f, "iterations %zu\nwall_seconds %a\nfinal_rrn %a\nfinal_residual_rel %a\n"
                        "terminated_by %d\nmethod %s\nalpha %a\nseed %llu\n"
                        "alpha_outside_bound %d\nskipped_zero_rows %zu\nx_rows %zu\nx_cols %zu\n"
                        "trace %zu\n",
                     rep.iterations, rep.wall_seconds, rep.final_rrn, rep.final_residual_rel,
                     rep.terminated_by == Terminated::Tolerance ? 0 : 1, rep.method_label.c_str(),
                     rep.alpha, (unsigned long long)rep.seed, rep.alpha_outside_bound ? 1 : 0,
                     rep.skipped_zero_rows, rep.X.rows(), rep.X.cols(), rep.trace.size());
        for (const auto& t : rep.trace)
            std::fprintf(f, "%zu %a %a %zu\n", t.k, t.rrn, t.residual_rel, t.selected_row);
        std::fclose(f);
    }
    std::vector<BenchmarkRow> rows(3);
    rows[0].problem_id = "gauss-500x100";
    rows[0].method = "grbk";
    rows[0].alpha_rule = "safe";
    rows[0].trials = 20;
    rows[0].it_mean = 13483.25;
    rows[0].it_std = 412.0625;
    rows[0].wall_mean_s = 0.1709;
    rows[0].speed_up_vs_rbk = 1.0 / 3.0;
    rows[1].problem_id = "ill \"conditioned\", κ=1e2";  // needs RFC-4180 quoting
    rows[1].method = "rgrbk";
    rows[1].theta = 0.25;
    rows[1].alpha_rule = "paper";
    rows[1].trials = 3;
    rows[1].it_mean = 1e6;
    rows[1].it_std = 0.0;
    rows[1].wall_mean_s = 2.5e-7;
    rows[1].failures = 3;
    rows[2].problem_id = "line\nbreak";
    rows[2].method = "rbk";
    rows[2].alpha_rule = "fixed";
    rows[2].trials = 1;
    rows[2].it_mean = 42.0;
    rows[2].wall_mean_s = 1e-300;
    rows[2].speed_up_vs_rbk = 1.0;
    write_text_file(dir + "/bench.csv", benchmark_to_csv(rows));
    write_text_file(dir + "/bench.json", benchmark_to_json(rows).dump(2) + "\n");
    std::vector<RestoreMetricsRow> rr(2);
    rr[0] = {"synthetic 256x256", "grbk", std::nullopt, 5000, 21.5, 30.125, 0.75, 0.9375};
    rr[1] = {"face,small", "rgrbk", 0.8, 123, 1.0 / 7.0, 33.7, 0.5, 0.939};
    write_text_file(dir + "/restore.csv", restore_metrics_to_csv(rr));
    std::printf("iterations=%zu trace=%zu\n", rep.iterations, rep.trace.size());
    return 0;
}
