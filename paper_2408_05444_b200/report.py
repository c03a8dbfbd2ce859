"""Report and trace formats of the reference, for drop-in CLIs.

Byte-compatible restatements of report.hpp:
  trace_to_csv            report.hpp:55-61   (RFC-4180, CRLF, %.17g, inf/-inf)
  benchmark_to_csv        report.hpp:63-75
  restore_metrics_to_csv  report.hpp:88-97
  solve_report_to_json    report.hpp:102-117 (+ "stop"/"tol" as axbsolve.cpp:208-209)
  benchmark_to_json       report.hpp:119-136
  dumps_json              nlohmann::json::dump(2): keys sorted, 2-space indent, UTF-8
                          unescaped, shortest round-trip doubles, "\\n" appended
Pinned byte for byte against the reference's own writers (tests/test_report.py,
fixtures from tests/golden/make_report_golden.cpp).
"""
from __future__ import annotations

import json
import math
import os
from typing import Iterable, Optional

from .solver import SolveReport, Terminated, TracePoint

TOOL_VERSION = "1.0.0"  # report.hpp:18


def _escape(field: str) -> str:  # report.hpp:25-34
    if not any(ch in field for ch in ',"\r\n'):
        return field
    return '"' + field.replace('"', '""') + '"'


def _num(v: float) -> str:  # report.hpp:36-41
    if math.isinf(v):
        return "inf" if v > 0 else "-inf"
    return "%.17g" % v


def _row(fields: Iterable[str]) -> str:  # report.hpp:43-50
    return ",".join(_escape(f) for f in fields) + "\r\n"


def trace_to_csv(trace: Iterable[TracePoint]) -> str:
    out = _row(["k", "rrn", "residual_rel", "row"])
    for t in trace:
        out += _row([str(t.k), _num(t.rrn), _num(t.residual_rel), str(t.selected_row)])
    return out


def benchmark_to_csv(rows) -> str:  # report.hpp:63-75
    out = _row(["problem_id", "method", "theta", "alpha_rule", "trials", "it_mean", "it_std",
                "wall_mean_s", "speed_up_vs_rbk", "failures"])
    for r in rows:
        out += _row([r.problem_id, r.method, "" if r.theta is None else _num(r.theta), r.alpha_rule,
                     str(r.trials), _num(r.it_mean), _num(r.it_std), _num(r.wall_mean_s),
                     "" if r.speed_up_vs_rbk is None else _num(r.speed_up_vs_rbk),
                     str(r.failures)])
    return out


def restore_metrics_to_csv(rows) -> str:  # report.hpp:88-97
    """rows: objects with image, method, theta (None or float), iterations,
    psnr_blurred, psnr_restored, ssim_blurred, ssim_restored."""
    out = _row(["image", "method", "theta", "iterations", "psnr_blurred", "psnr_restored",
                "ssim_blurred", "ssim_restored"])
    for r in rows:
        out += _row([r.image, r.method, "" if r.theta is None else _num(r.theta), str(r.iterations),
                     _num(r.psnr_blurred), _num(r.psnr_restored), _num(r.ssim_blurred),
                     _num(r.ssim_restored)])
    return out


def benchmark_to_json(rows) -> list:  # report.hpp:119-136
    out = []
    for r in rows:
        j = {"problem_id": r.problem_id, "method": r.method}
        if r.theta is not None:
            j["theta"] = float(r.theta)
        j.update({"alpha_rule": r.alpha_rule, "trials": int(r.trials), "it_mean": float(r.it_mean),
                  "it_std": float(r.it_std), "wall_mean_s": float(r.wall_mean_s)})
        if r.speed_up_vs_rbk is not None:
            j["speed_up_vs_rbk"] = float(r.speed_up_vs_rbk)
        j["failures"] = int(r.failures)
        out.append(j)
    return out


def solve_report_to_json(rep: SolveReport, stop: Optional[str] = None,
                         tol: Optional[float] = None) -> dict:
    j = {
        "iterations": int(rep.iterations),
        "wall_seconds": float(rep.wall_seconds),
        "final_rrn": float(rep.final_rrn),
        "final_residual_rel": float(rep.final_residual_rel),
        "terminated_by": "tolerance" if rep.terminated_by == Terminated.Tolerance else "max_iter",
        "method": rep.method_label,
        "alpha": float(rep.alpha),
        "seed": int(rep.seed),
        "alpha_outside_bound": bool(rep.alpha_outside_bound),
        "skipped_zero_rows": int(rep.skipped_zero_rows),
        "x_rows": int(rep.X.shape[0]) if rep.X is not None else 0,
        "x_cols": int(rep.X.shape[1]) if rep.X is not None else 0,
    }
    if stop is not None:
        j["stop"] = stop
    if tol is not None:
        j["tol"] = float(tol)
    return j


def dumps_json(obj) -> str:
    """nlohmann::json::dump(2) + "\\n" (axbsolve.cpp:210): std::map key order,
    UTF-8 left unescaped, doubles shortest round-trip ("1000000.0", "2.5e-07")."""
    return json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False) + "\n"


def write_solve_outputs(out_dir: str, rep: SolveReport, stop: str, tol: float,
                        trace: bool = True) -> None:
    """report.json (+ trace.csv) as `axbsolve solve` writes them (axbsolve.cpp:205-212)."""
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "report.json"), "w", newline="", encoding="utf-8") as f:
        f.write(dumps_json(solve_report_to_json(rep, stop, tol)))
    if trace:
        with open(os.path.join(out_dir, "trace.csv"), "w", newline="") as f:
            f.write(trace_to_csv(rep.trace))
