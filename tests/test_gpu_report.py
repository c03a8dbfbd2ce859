"""GPU: report / trace outputs of a device run.

The `axbsolve solve` replay contract (cli_tests.cpp:168-195): the same solve run
twice writes byte-identical trace.csv and the same report.json apart from the
wall time.  And the device run's trace against the REFERENCE's own trace.csv for
the same config-1 run (tests/golden/report/, written by report.hpp through
tests/golden/make_report_golden.cpp): the same selected rows and k column up to
where the shorter run stops, the reference's CSV layout, a stop within ±2
iterations (fresh vs running sums).
"""
import gzip
import json
import os

import numpy as np
import pytest

import oracle_lib as O
from paper_2408_05444_b200 import report

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "report")


def _csv_rows(text):
    lines = text.split("\r\n")
    assert lines[-1] == ""
    return [ln.split(",") for ln in lines[:-1]]


def test_device_run_replays_and_matches_reference_trace(axb, orc, tmp_path):
    A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)

    def solve(out):
        cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-12, X),
                              max_iter=10 ** 6, seed=42, record_trace=True)
        rep = axb.solve(A, B, Cm, None, cfg)
        report.write_solve_outputs(str(out), rep, "rrn", 1e-12)
        return rep

    r1, r2 = solve(tmp_path / "s1"), solve(tmp_path / "s2")
    t1 = open(tmp_path / "s1" / "trace.csv", "rb").read()
    assert t1 == open(tmp_path / "s2" / "trace.csv", "rb").read()
    j1 = json.load(open(tmp_path / "s1" / "report.json"))
    j2 = json.load(open(tmp_path / "s2" / "report.json"))
    j1.pop("wall_seconds"), j2.pop("wall_seconds")
    assert j1 == j2 and j1["terminated_by"] == "tolerance" and j1["final_rrn"] <= 1e-12
    with gzip.open(os.path.join(GOLD, "trace.csv.gz"), "rb") as f:
        ref = _csv_rows(f.read().decode())
    dev = _csv_rows(t1.decode())
    assert dev[0] == ref[0] == ["k", "rrn", "residual_rel", "row"]
    nc = min(len(ref), len(dev)) - 1
    assert nc > 10000
    assert [r[0] for r in dev[1:nc + 1]] == [r[0] for r in ref[1:nc + 1]]  # k, decimated past 10⁴
    assert [r[3] for r in dev[1:nc + 1]] == [r[3] for r in ref[1:nc + 1]]  # the selected rows
    rr = np.array([float(r[1]) for r in ref[1:nc + 1]])
    dr = np.array([float(r[1]) for r in dev[1:nc + 1]])
    assert np.max(np.abs(dr - rr) / rr) <= 1e-6
    ref_json = json.load(open(os.path.join(GOLD, "report.json")))
    assert abs(j1["iterations"] - ref_json["iterations"]) <= 2
    assert j1["alpha"] == ref_json["alpha"] and j1["method"] == ref_json["method"]
