"""CPU: report / trace formats (report.hpp:55-117, schemas/solve_report.schema.json)."""
import json
import os

import numpy as np

from paper_2408_05444_b200 import report
from paper_2408_05444_b200.solver import SolveReport, Terminated, TracePoint

SCHEMA = {
    "required": ["iterations", "wall_seconds", "final_rrn", "final_residual_rel", "terminated_by",
                 "method", "alpha", "seed"],
    "enums": {"terminated_by": {"tolerance", "max_iter"},
              "method": {"bk", "rbk", "grbk", "rgrbk", "mwrbk"}, "stop": {"rrn", "residual"}},
}


def make_rep():
    return SolveReport(iterations=3, wall_seconds=0.25, final_rrn=1e-13, final_residual_rel=2.5e-7,
                       terminated_by=Terminated.Tolerance,
                       trace=[TracePoint(0, 0.5, 0.25, 7), TracePoint(1, float("inf"), 1 / 3, 2)],
                       X=np.zeros((4, 5)), alpha=1.0 / 3.0, seed=42, method_label="grbk")


def test_trace_csv_format():
    csv = report.trace_to_csv(make_rep().trace)
    assert csv == ("k,rrn,residual_rel,row\r\n0,0.5,0.25,7\r\n"
                   "1,inf,0.33333333333333331,2\r\n")


def test_report_json_matches_schema_and_nlohmann_layout(tmp_path):
    rep = make_rep()
    report.write_solve_outputs(str(tmp_path), rep, "rrn", 1e-12)
    text = open(os.path.join(tmp_path, "report.json")).read()
    j = json.loads(text)
    for k in SCHEMA["required"]:
        assert k in j
    for k, allowed in SCHEMA["enums"].items():
        assert j[k] in allowed
    assert list(j) == sorted(j)  # nlohmann's std::map key order
    assert text.endswith("}\n") and '\n  "alpha": 0.3333333333333333,\n' in text
    assert (j["x_rows"], j["x_cols"], j["tol"]) == (4, 5, 1e-12)
    assert open(os.path.join(tmp_path, "trace.csv"), newline="").read().startswith("k,rrn")


def test_csv_escaping():
    assert report._escape('a"b,c') == '"a""b,c"'
    assert report._escape("plain") == "plain"


def test_substream_seeds_match_reference_golden():
    """pool.substream_seed == RngStream(seed).substream(t).seed() (rng.hpp:102-104)."""
    from paper_2408_05444_b200 import pool

    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "rng.npz"))
    for i, sd in enumerate(g["seeds"]):
        for t in range(4):
            assert pool.substream_seed(int(sd), t) == int(g["substream_seeds"][i][t])


def test_benchmark_csv_layout():
    from paper_2408_05444_b200.pool import BenchmarkRow

    rows = [BenchmarkRow("p1", "rbk", None, "safe", 3, 10.0, 1.0, 0.5, 1.0, 0),
            BenchmarkRow("p1", "rgrbk", 0.5, "safe", 3, 5.0, 0.0, 0.25, 2.0, 1)]
    csv = report.benchmark_to_csv(rows)
    assert csv.splitlines()[0] == ("problem_id,method,theta,alpha_rule,trials,it_mean,it_std,"
                                   "wall_mean_s,speed_up_vs_rbk,failures")
    assert csv.splitlines()[2] == "p1,rgrbk,0.5,safe,3,5,0,0.25,2,1"


# ---- pinned byte for byte against the reference's own writers -------------
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "report")


def _read(name):
    import gzip

    path = os.path.join(GOLD, name)
    if name.endswith(".gz"):
        with gzip.open(path, "rb") as f:
            return f.read().decode("utf-8")
    with open(path, "rb") as f:
        return f.read().decode("utf-8")


def _reference_run():
    """The reference's SolveReport + trace for a config-1 run (run_raw.txt: hex floats
    written by tests/golden/make_report_golden.cpp)."""
    lines = _read("run_raw.txt.gz").splitlines()
    kv = {}
    i = 0
    while not lines[i].startswith("trace "):
        k, v = lines[i].split(" ", 1)
        kv[k] = v
        i += 1
    nt = int(lines[i].split()[1])
    trace = []
    for ln in lines[i + 1:i + 1 + nt]:
        k, rrn, rel, row = ln.split()
        trace.append(TracePoint(int(k), float.fromhex(rrn), float.fromhex(rel), int(row)))
    rep = SolveReport(iterations=int(kv["iterations"]), wall_seconds=float.fromhex(kv["wall_seconds"]),
                      final_rrn=float.fromhex(kv["final_rrn"]),
                      final_residual_rel=float.fromhex(kv["final_residual_rel"]),
                      terminated_by=Terminated(int(kv["terminated_by"])), trace=trace,
                      X=np.zeros((int(kv["x_rows"]), int(kv["x_cols"]))),
                      alpha=float.fromhex(kv["alpha"]), seed=int(kv["seed"]),
                      method_label=kv["method"],
                      alpha_outside_bound=bool(int(kv["alpha_outside_bound"])),
                      skipped_zero_rows=int(kv["skipped_zero_rows"]))
    return rep


def test_trace_and_report_json_byte_identical_to_reference(tmp_path):
    """report.hpp:55-61 trace_to_csv and :102-117 solve_report_to_json + the CLI's
    stop/tol keys dumped with dump(2) (axbsolve.cpp:207-212), fed the reference's
    own config-1 run (13,483 GRBK iterations, 10,349 trace points across the
    10⁴ decimation boundary): identical bytes."""
    rep = _reference_run()
    assert len(rep.trace) == 10349 and rep.iterations == 13483
    assert report.trace_to_csv(rep.trace) == _read("trace.csv.gz")
    assert report.dumps_json(report.solve_report_to_json(rep, "rrn", 1e-12)) == _read("report.json")
    report.write_solve_outputs(str(tmp_path), rep, "rrn", 1e-12)
    with open(os.path.join(tmp_path, "report.json"), "rb") as f:
        assert f.read() == _read("report.json").encode("utf-8")
    with open(os.path.join(tmp_path, "trace.csv"), "rb") as f:
        assert f.read() == _read("trace.csv.gz").encode("utf-8")


def test_benchmark_and_restore_formats_byte_identical_to_reference():
    """report.hpp:63-75, :88-97, :119-136 on rows with optional θ / speed-up and
    fields that need RFC-4180 quoting (comma, quote, newline, UTF-8)."""
    from types import SimpleNamespace

    from paper_2408_05444_b200.pool import BenchmarkRow

    rows = [BenchmarkRow("gauss-500x100", "grbk", None, "safe", 20, 13483.25, 412.0625, 0.1709,
                         1.0 / 3.0, 0),
            BenchmarkRow('ill "conditioned", κ=1e2', "rgrbk", 0.25, "paper", 3, 1e6, 0.0, 2.5e-7,
                         None, 3),
            BenchmarkRow("line\nbreak", "rbk", None, "fixed", 1, 42.0, 0.0, 1e-300, 1.0, 0)]
    assert report.benchmark_to_csv(rows) == _read("bench.csv")
    assert report.dumps_json(report.benchmark_to_json(rows)) == _read("bench.json")
    rr = [SimpleNamespace(image="synthetic 256x256", method="grbk", theta=None, iterations=5000,
                          psnr_blurred=21.5, psnr_restored=30.125, ssim_blurred=0.75,
                          ssim_restored=0.9375),
          SimpleNamespace(image="face,small", method="rgrbk", theta=0.8, iterations=123,
                          psnr_blurred=1.0 / 7.0, psnr_restored=33.7, ssim_blurred=0.5,
                          ssim_restored=0.939)]
    assert report.restore_metrics_to_csv(rr) == _read("restore.csv")
