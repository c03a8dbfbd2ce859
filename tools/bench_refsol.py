#!/usr/bin/env python3
"""Time the device reference solution at BASELINE config-3 sizes.

Device: P.reference_solution on A 8192×2048 · B 2048×8192 Gaussian (unique X*),
reporting Jacobi sweeps and the device time (CUDA events, inputs resident) and
the wall time including host↔device copies.  CPU: the reference's own svd
(oracle/_ref, one thread) on a bounded sample, extrapolated by the Jacobi cost
model pairs·m·sweeps (n(n−1)/2 pairs of length-m columns per sweep) — running it
at full size would take hours.

    python tools/bench_refsol.py [--m 8192 --p 2048] [--sample 1024x256]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=8192)
    ap.add_argument("--p", type=int, default=2048)
    ap.add_argument("--sample", default="1024x256")
    ap.add_argument("--repeat", type=int, default=2)
    args = ap.parse_args()
    import paper_2408_05444_b200 as P

    rng = np.random.default_rng(8)
    m, p = args.m, args.p
    q, n = p, m
    A = rng.standard_normal((m, p))
    B = rng.standard_normal((q, n))
    Xs = rng.standard_normal((p, q))
    Cm = (A @ Xs) @ B
    out = {"config": f"A {m}x{p}, B {q}x{n}, Gaussian, unique X*"}
    best = None
    for _ in range(args.repeat):
        t0 = time.perf_counter()
        r = P.reference_solution(A, B, Cm)
        wall = time.perf_counter() - t0
        sa, sb, ms = P.analysis.last_stats()
        if best is None or ms < best[2]:
            best = (sa, sb, ms, wall)
    sa, sb, ms, wall = best
    out.update({"sweeps": [sa, sb], "device_ms": ms, "wall_s": wall,
                "rel_err_vs_generator": float(np.linalg.norm(r.X_star - Xs) / np.linalg.norm(Xs)),
                "kind": r.kind.name})
    rounds = (sa + sb) * (p - 1 + (p & 1))
    out["us_per_round"] = ms * 1e3 / rounds
    # algorithmic bytes of one round: W read twice (dots, rotate) + written once,
    # V read + written — the first pass is the only one that must come from HBM
    w_bytes, v_bytes = 8.0 * m * p, 8.0 * p * p
    out["round_hbm_GBps"] = (2 * w_bytes + 2 * v_bytes) / (ms * 1e-3 / rounds) / 1e9
    try:
        import oracle_lib as O
        if O.ref_available():
            sm, sn = map(int, args.sample.split("x"))
            M = rng.standard_normal((sm, sn))
            an = O.Analysis(O.ref())
            t0 = time.perf_counter()
            an.svd(M)
            cpu = time.perf_counter() - t0
            # sweeps at the sample: count via the restatement's cap trick is not
            # exposed; use the device's sweep count on the same sample instead
            f = P.svd(M, compute_uv=False)
            s_sweeps = P.analysis.last_stats()[0]
            per = cpu / (sn * (sn - 1) / 2 * sm * s_sweeps)
            est = per * (p * (p - 1) / 2 * m) * (sa + sb)
            out["cpu_reference"] = {"kind": "reference", "cores": 1,
                                    "sample": f"svd of a {sm}x{sn} Gaussian ({s_sweeps} sweeps)",
                                    "sample_s": cpu, "s_per_pair_elem": per,
                                    "extrapolated_svd_s": est,
                                    "note": "both SVDs at full size, Jacobi cost model"}
            del f
    except Exception as e:  # noqa: BLE001
        out["cpu_reference"] = {"unavailable": str(e)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
