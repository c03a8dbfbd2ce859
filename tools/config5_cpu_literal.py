"""Checks the reference arm's ×64 extrapolation for BASELINE config 5 once, at the
literal size, on the GPU box's host (test infrastructure; no GPU is used).

bench.py --impl reference cannot construct config 5 (65536×8192 · 8192×32768)
through the reference engine: its constructor would form G = A·Aᵀ (34 GB) and
BᵀB (8.6 GB) with ~10¹⁴ single-threaded FLOP.  It runs the 1/8-per-dimension
instance instead and divides the rate by 64, because every per-iteration term of
the reference's step() (R update m·n, z = BᵀB·R_iᵀ n², y q·n, X p·q) shrinks by
exactly 8² there.  This tool measures the reference's per-iteration algorithm at
BOTH sizes with the same engine — the bitwise-equal C port (oracle/axb_oracle.c)
driven over precomputed constructor caches (C, G, BᵀB formed with the host's
multithreaded BLAS, setup only) — and reports the measured ratio next to 64.

    python tools/config5_cpu_literal.py [--steps 3] [--small-steps 200]
Needs ~110 GB of host RAM; prints one JSON line.
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


def instance(m, p, q, n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, p)) * p ** -0.5
    B = rng.standard_normal((q, n)) * n ** -0.5
    Xs = rng.standard_normal((p, q))
    return A, B, Xs


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def per_iteration_s(orc, m, p, q, n, steps, seed):
    t0 = time.perf_counter()
    A, B, Xs = instance(m, p, q, n, seed)
    log(f"[{m}x{p}.{q}x{n}] inputs {time.perf_counter() - t0:.1f}s")
    # products in row blocks: the host BLAS takes 32-bit dimensions and element
    # counts (a one-call 65536×65536 result overflows them and crashes)
    blk = 4096
    T = A @ Xs
    C = np.empty((m, n))
    for i0 in range(0, m, blk):
        C[i0:i0 + blk] = T[i0:i0 + blk] @ B
    del T
    log(f"  C {time.perf_counter() - t0:.1f}s")
    G = np.empty((m, m))
    At = np.ascontiguousarray(A.T)
    for i0 in range(0, m, blk):
        G[i0:i0 + blk] = A[i0:i0 + blk] @ At
    del At
    log(f"  G {time.perf_counter() - t0:.1f}s")
    BtB = B.T @ B
    log(f"  BtB {time.perf_counter() - t0:.1f}s")
    v = np.ones(q) / np.sqrt(q)  # ‖B‖₂² by a short power iteration on B·Bᵀ (timing only)
    for _ in range(60):
        w = B @ (B.T @ v)
        lam = float(np.linalg.norm(w))
        v = w / lam
    alpha = 1.0 / lam
    setup = time.perf_counter() - t0
    cfg = O.make_config(method=O.GRBK, stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=Xs, seed=42,
                        refresh_interval=0, max_iter=10 ** 9)
    s = O.PreparedSolver(orc, A, B, C, np.zeros((p, q)), C, G, BtB, alpha, cfg)
    log(f"  prepared {time.perf_counter() - t0:.1f}s")
    s.steps(1)  # warm
    t0 = time.perf_counter()
    s.steps(steps)
    dt = (time.perf_counter() - t0) / steps
    del s
    return dt, setup


def main():
    import faulthandler

    faulthandler.enable()
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--small-steps", type=int, default=200)
    args = ap.parse_args()
    try:
        import psutil

        avail = psutil.virtual_memory().available
    except Exception:
        avail = 0
    orc = O.oracle()
    small, small_setup = per_iteration_s(orc, 8192, 1024, 1024, 4096, args.small_steps, 7)
    out = {"tool": "config5_cpu_literal", "engine": "oracle C port of solver.hpp step() (bitwise "
           "the reference's per-iteration algorithm), 1 thread",
           "small_instance": "8192x1024.1024x4096", "small_s_per_iter": small,
           "host_available_gb": round(avail / 1e9, 1)}
    if avail and avail < 115e9:
        out["literal"] = f"skipped: {avail / 1e9:.0f} GB available, ~110 GB needed"
    else:
        big, big_setup = per_iteration_s(orc, 65536, 8192, 8192, 32768, args.steps, 7)
        out.update({"literal_instance": "65536x8192.8192x32768", "literal_s_per_iter": big,
                    "literal_setup_s": round(big_setup, 1), "measured_ratio": big / small,
                    "extrapolation_factor": 64,
                    "extrapolated_it_per_s": 1.0 / (64 * small), "literal_it_per_s": 1.0 / big})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
