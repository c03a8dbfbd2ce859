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
