"""BASELINE config 2 at its full budget: 10⁴ deterministic ME-MWRBK steps (and 10⁴
self-selected ME-GRBK steps) on the device against the unmodified reference engine
(oracle/_ref, the reference headers compiled in place) and the C oracle, all on the
same inputs; the index sequences are compared element-wise and X, R at step 10⁴
relative to the reference's.  Test infrastructure: the reference and
the oracle are the checkers here, the device path is the thing checked.

A 2000×500 = U·diag(σ)·Vᵀ, B 400×2000 the same way, σ log-spaced 1..1e-2 (κ = 100),
X* N(0,1), C = A·X*·B (tests/configs.py:config2).

    python tools/config2_sequence.py [--steps 10000] [--seed 2]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import configs  # noqa: E402
import oracle_lib as O  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--seed", type=int, default=2)
    args = ap.parse_args()
    import paper_2408_05444_b200 as axb

    A, B, Xs, Cm = configs.config2(seed=args.seed)
    K = args.steps
    checkers = {"oracle": O.oracle()}
    if O.ref_available():
        checkers["reference"] = O.ref()
    runs = [("MWRBK", O.MWRBK, axb.Method.mwrbk()), ("GRBK", O.GRBK, axb.Method.grbk())]

    # the CPU checkers in parallel threads (ctypes drops the GIL)
    res = {}

    def cpu(name, lib, label, tag):
        cfg = O.make_config(method=tag, seed=42, max_iter=10 ** 9, refresh_interval=0,
                            stop_kind=O.SOLUTION_RRN, tol=0.0, reference=Xs)
        s = O.Solver(lib, A, B, Cm, None, cfg)
        t0 = time.perf_counter()
        rows = s.steps(K)
        res[(name, label)] = (rows, s.X(), s.R(), time.perf_counter() - t0, s.alpha)

    th = [threading.Thread(target=cpu, args=(n, lib, label, tag))
          for n, lib in checkers.items() for label, tag, _ in runs]
    for t in th:
        t.start()

    dev = {}
    for path in ("default", "graph"):
        if path == "graph":
            os.environ["AXB_PERSIST"] = "0"
        for label, _, meth in runs:
            cfg = axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(0.0, Xs),
                                  max_iter=10 ** 9, seed=42, refresh_interval=0)
            s = axb.Solver(A, B, Cm, None, cfg)
            t0 = time.perf_counter()
            rows = s.steps(K)
            dev[(path, label)] = (rows, s.X(), s.R(), time.perf_counter() - t0, s.alpha())
        os.environ.pop("AXB_PERSIST", None)
    for t in th:
        t.join()

    err0 = None
    for (path, label), (rows, X, R, secs, alpha) in dev.items():
        for name in checkers:
            rrows, rX, rR, rsecs, ralpha = res[(name, label)]
            mism = np.nonzero(rows.astype(np.uint64) != rrows)[0]
            out = {"config": "config2 A 2000x500, B 400x2000, kappa 100 each", "method": label,
                   "device_path": path, "checker": name, "steps": K,
                   "index_mismatches": int(mism.size),
                   "first_mismatch": int(mism[0]) if mism.size else None,
                   "alpha_identical": alpha == ralpha,
                   "X_rel_diff": rel(X, rX), "R_rel_diff": rel(R, rR),
                   "err_device": rel(X, Xs), "err_checker": rel(rX, Xs),
                   "device_seconds": round(secs, 3), "checker_seconds_1core": round(rsecs, 1)}
            print(json.dumps(out), flush=True)
            if out["index_mismatches"] or out["X_rel_diff"] > 1e-10:
                err0 = 1
    sys.exit(err0 or 0)


if __name__ == "__main__":
    main()
