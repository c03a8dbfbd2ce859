"""BASELINE config 4 at full size (1024×1024 blur channels) against the oracle.

The reference constructor cannot run it: its spectral_norm(B) (tol 1e-10, cap 5000,
decomp.hpp:207-239, solver.hpp:168) throws ConvergenceError for the 1024-wide blur
(SURVEY §8(c)(i)).  As SURVEY prescribes, the checker is the C restatement of the
reference's per-iteration algorithm (oracle/, bitwise-pinned to the reference at the
sizes the reference can run) with α = 1/‖B‖₂² from the reference's power iteration
with a raised cap (orc_spectral_norm(B, 1e-10, 200000)); the device gets the same
cap (Options.spectral_max_iter), so α must agree bit for bit.  Test infrastructure:
the oracle checks, the device path is checked.

Per channel and half-band (7 and 15, both readings of 'bandwidth 15'), MWRBK and
self-selected GRBK: index sequences over K steps compared element-wise, X and R at
step K relative to the oracle's, and the residual/PSNR each reaches.

    python tools/config4_parity.py [--steps 3000]
"""
import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402
from bench import CONFIGS, make_channel, psnr  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3000)
    args = ap.parse_args()
    import paper_2408_05444_b200 as axb

    orc = O.oracle()
    K = args.steps
    cases = []
    for hb in (7, 15):
        cfg = dict(CONFIGS[4], half_band=hb)
        spec = None
        for c in range(cfg["channels"]):
            A, B, Cm, Xs = make_channel(cfg, 4, c)
            if spec is None:  # B is the same blur for every channel
                st = C.c_int()
                spec = orc.spectral_norm(O._ptr(np.ascontiguousarray(B)), B.shape[0], B.shape[1],
                                         1e-10, 200000, C.byref(st), None)
                assert st.value == 0
            for label, tag, meth in (("MWRBK", O.MWRBK, axb.Method.mwrbk()),
                                     ("GRBK", O.GRBK, axb.Method.grbk())):
                cases.append(dict(hb=hb, c=c, A=A, B=B, Cm=Cm, Xs=Xs, alpha=1.0 / (spec * spec),
                                  label=label, tag=tag, meth=meth))

    res = [None] * len(cases)

    def cpu(i):
        k = cases[i]
        cfg_o = O.make_config(method=k["tag"], seed=42, max_iter=10 ** 9, refresh_interval=0,
                              stop_kind=O.RESIDUAL_REL, tol=0.0)
        s = O.PreparedSolver(orc, k["A"], k["B"], k["Cm"], np.zeros_like(k["Xs"]), k["Cm"],
                             k["A"] @ k["A"].T, k["B"].T @ k["B"], k["alpha"], cfg_o)
        t0 = time.perf_counter()
        rows = s.steps(K)
        res[i] = (rows, s.X(), s.R(), time.perf_counter() - t0)

    th = [threading.Thread(target=cpu, args=(i,)) for i in range(len(cases))]
    for t in th:
        t.start()
    dev = []
    for k in cases:
        cfg = axb.SolveConfig(method=k["meth"], stop=axb.StopRule.residual_rel(0.0),
                              max_iter=10 ** 9, seed=42, refresh_interval=0)
        s = axb.Solver(k["A"], k["B"], k["Cm"], None, cfg, axb.Options(spectral_max_iter=200000))
        t0 = time.perf_counter()
        rows = s.steps(K)
        dev.append((rows, s.X(), s.R(), time.perf_counter() - t0, s.alpha()))
        del s
    for t in th:
        t.join()
    bad = 0
    for k, (rows, X, R, secs, alpha), (orows, oX, oR, osecs) in zip(cases, dev, res):
        mism = np.nonzero(rows.astype(np.uint64) != orows)[0]
        out = {"config": f"config4 channel {k['c']} 1024x1024 blur, half-band {k['hb']}",
               "method": k["label"], "steps": K, "index_mismatches": int(mism.size),
               "first_mismatch": int(mism[0]) if mism.size else None,
               "alpha_identical": alpha == k["alpha"],
               "X_rel_diff": rel(X, oX), "R_rel_diff": rel(R, oR),
               "residual_rel_device": float(np.linalg.norm(R) / np.linalg.norm(k["Cm"])),
               "residual_rel_oracle": float(np.linalg.norm(oR) / np.linalg.norm(k["Cm"])),
               "psnr_db_device": psnr([k["Xs"]], [X]), "psnr_db_oracle": psnr([k["Xs"]], [oX]),
               "device_seconds": round(secs, 3), "oracle_seconds_1core": round(osecs, 1)}
        print(json.dumps(out), flush=True)
        bad |= bool(mism.size) or out["X_rel_diff"] > 1e-10 or not out["alpha_identical"]
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
