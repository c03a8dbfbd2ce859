"""BASELINE config 5 at its LITERAL size against the CPU oracle (on the GPU box's host).

SURVEY §8(c)(ii) put config 5 out of the oracle's reach (≈84 GB of host state); the
pool's boxes have 196 GB, so this tool runs it once: A 65536×8192 N(0,1/8192),
B 8192×32768 N(0,1/32768), X* N(0,1), C = A·X*·B, X0 = 0, ME-GRBK.

  cpu   the oracle's C port of solver.hpp step() (bitwise the reference's
        per-iteration algorithm) over constructor caches formed with the host BLAS
        (C, G = A·Aᵀ, BᵀB: ~10¹⁴ FLOP that the reference's sequential constructor
        cannot do in a session) — one core, ~3.7 s per iteration
  gpu   the same host arrays through the C-ABI (single GPU; α from the device's
        power iteration is handed to the CPU side so both use the same value)

Prints one JSON line: the selected rows of both, the first mismatch, X and ‖R_l‖²
relative differences.  Needs ~95 GB of host RAM and ~8 minutes.

    python tools/config5_literal_parity.py [--steps 24] [--method grbk|mwrbk|rgrbk025|rgrbk075]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    import faulthandler

    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--method", default="grbk", choices=["grbk", "mwrbk", "rgrbk025", "rgrbk075"])
    ap.add_argument("--scale", type=int, default=1, help="divide every dimension (smoke test of the tool)")
    args = ap.parse_args()
    d = args.scale
    m, p, q, n = 65536 // d, 8192 // d, 8192 // d, 32768 // d
    import paper_2408_05444_b200 as axb

    t0 = time.perf_counter()
    rng = np.random.default_rng(7)
    A = rng.standard_normal((m, p)) * p ** -0.5
    B = rng.standard_normal((q, n)) * n ** -0.5
    Xs = rng.standard_normal((p, q))
    blk = 4096  # host BLAS takes 32-bit element counts: products in row blocks
    T = A @ Xs
    C = np.empty((m, n))
    for i0 in range(0, m, blk):
        C[i0:i0 + blk] = T[i0:i0 + blk] @ B
    del T
    log(f"inputs and C {time.perf_counter() - t0:.0f}s")

    meth, tag, theta = {"grbk": (axb.Method.grbk(), O.GRBK, None), "mwrbk": (axb.Method.mwrbk(), O.MWRBK, None),
                        "rgrbk025": (axb.Method.rgrbk(0.25), O.RGRBK, 0.25),
                        "rgrbk075": (axb.Method.rgrbk(0.75), O.RGRBK, 0.75)}[args.method]
    cfg = axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(0.0, Xs), seed=42,
                          refresh_interval=0, max_iter=10 ** 9)
    s = axb.Solver(A, B, C, None, cfg, axb.Options(spectral_max_iter=200000, cache_gram=1))
    alpha = s.alpha()
    t1 = time.perf_counter()
    rows_g = s.steps(args.steps)
    gpu_s = time.perf_counter() - t1
    Xg, rsq_g = s.X(), s.residual_row_sq()
    del s
    log(f"device: alpha {alpha:.6e}, {args.steps} steps in {gpu_s:.2f}s")

    G = np.empty((m, m))
    At = np.ascontiguousarray(A.T)
    for i0 in range(0, m, blk):
        G[i0:i0 + blk] = A[i0:i0 + blk] @ At
    del At
    BtB = B.T @ B
    log(f"G, BtB {time.perf_counter() - t0:.0f}s")
    orc = O.oracle()
    cfg_o = O.make_config(method=tag, theta=theta, stop_kind=O.SOLUTION_RRN, tol=0.0, reference=Xs, seed=42,
                          refresh_interval=0, max_iter=10 ** 9)
    so = O.PreparedSolver(orc, A, B, C, np.zeros((p, q)), C, G, BtB, alpha, cfg_o)
    t1 = time.perf_counter()
    rows_c = so.steps(args.steps)
    cpu_s = time.perf_counter() - t1
    Xc = so.X()
    rsq_c = np.empty(m)
    so.lib.get_r_sq(so.h, O._ptr(rsq_c))
    log(f"oracle: {args.steps} steps in {cpu_s:.1f}s")
    rows_g = np.asarray(rows_g, dtype=np.int64)
    rows_c = np.asarray(rows_c, dtype=np.int64)
    mism = np.nonzero(rows_g != rows_c)[0]
    out = {"tool": "config5_literal_parity", "instance": f"{m}x{p}.{q}x{n}", "method": args.method, "steps": args.steps,
           "alpha": alpha, "rows_device": rows_g.tolist(), "rows_oracle": rows_c.tolist(),
           "index_mismatches": int(mism.size), "first_mismatch": int(mism[0]) if mism.size else None,
           "X_rel_diff": float(np.linalg.norm(Xg - Xc) / max(np.linalg.norm(Xc), 1e-300)),
           "r_sq_rel_diff": float(np.max(np.abs(rsq_g - rsq_c) / np.maximum(rsq_c, 1e-300))),
           "device_seconds": round(gpu_s, 3), "oracle_seconds_1core": round(cpu_s, 1),
           "checker": "oracle C port of solver.hpp step() over host-BLAS constructor caches (G, BtB, C)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
