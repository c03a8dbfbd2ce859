"""BASELINE config 3 at FULL size pinned against the UNMODIFIED reference engine.

A 8192×2048 · B 2048×8192 iid N(0,1), X* 2048×2048 N(0,1), X0 N(0,1), C = A·X*·B.
Two sides, one fixture:

  ref  (this container, needs oracle/_ref/libaxbref.so): the inputs are drawn with
       the reference's own RngStream restated in oracle/ (generate()'s substreams
       1/2/3 for A, B, X*, problems.hpp:346-349; substream 4 for X0), C is formed
       with the reference's sequential ikj matmul (matrix.hpp:325-338, restated in
       oracle/axb_oracle.c, rows split over host threads — bitwise the same on any
       x86-64 host because each row's k-order is fixed and fp-contract is off).
       Each variant then runs through the unmodified axb::Solver (its constructor:
       ‖B‖₂ power iteration, G = A·Aᵀ, BᵀB, R0; then STEPS step() calls), and the
       fixture tests/golden/config3_pin.npz keeps: the selected rows, α, ‖X‖²_F,
       ‖X − X0‖²_F, 8 sampled rows of X, 16 bilinear probes uᵀXv, and r_sq.
  gpu  (a B200): the same inputs (same restated generator, same threaded matmul),
       then the device solver through the C-ABI with the reference's α
       (Options.alpha_override; SURVEY §7 "pass the oracle's α"): (i) self-selected rows must equal the
       reference's, (ii) a replay of the reference's rows must give X within 1e-10
       (relative, on every stored digest) and r_sq within 1e-9.

Variants: ME-GRBK (θ=½), ME-RGRBK θ=0.25 and 0.75, ME-MWRBK, and the rank-deficient
system: A = A1·A2/√1536 with A1 8192×1536, A2 1536×2048 N(0,1) (substreams 5, 6),
so rank(A) = 1536 exactly.  (BASELINE words it as "zeroing singular values"; a
factor product gives the same rank without an SVD whose bits would depend on the
host's LAPACK, which the two sides must not.)

    python tools/config3_pin.py ref [--steps 500] [--threads 8]
    python tools/config3_pin.py gpu [--threads 16]    # on the B200; prints JSON lines
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402

FIXTURE = os.path.join(ROOT, "tests", "golden", "config3_pin.npz")
M, P, Q, N = 8192, 2048, 2048, 8192
RANK = 1536
ROOT_SEED = 3
SOLVER_SEED = 42
VARIANTS = [  # name, method, theta, system
    ("grbk", O.GRBK, None, "full"),
    ("rgrbk025", O.RGRBK, 0.25, "full"),
    ("rgrbk075", O.RGRBK, 0.75, "full"),
    ("mwrbk", O.MWRBK, None, "full"),
    ("rankdef_grbk", O.GRBK, None, "rankdef"),
]
SAMPLE_ROWS = np.array([0, 1, 511, 1024, 1337, 1536, 2046, 2047])
N_PROBES = 16

_dp = C.POINTER(C.c_double)


def _p(a):
    return a.ctypes.data_as(_dp)


def _orc():
    lib = O.oracle()
    S = C.c_size_t
    lib.matmul = lib._f("matmul", None, [_dp, S, S, _dp, S, _dp])
    lib.dense_gaussian = lib._f("dense_gaussian", None, [C.c_void_p, S, S, _dp])
    return lib


def gaussian(lib, sub, rows, cols):
    """RngStream(ROOT_SEED).substream(sub) → dense_gaussian (rng.hpp:102-104, 126-131)."""
    root, s = O.Rng(), O.Rng()
    lib.rng_init(C.byref(root), ROOT_SEED)
    lib.rng_substream(C.byref(root), sub, C.byref(s))
    out = np.empty((rows, cols))
    lib.dense_gaussian(C.byref(s), rows, cols, _p(out))
    return out


def matmul_mt(lib, a, b, threads):
    """matrix.hpp:325-338 (ikj, exact zeros skipped) with rows split over threads:
    every output row is computed by the same sequential loop, so the result is
    bitwise orc_matmul's (ctypes drops the GIL during the call)."""
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    ar, ac = a.shape
    bc = b.shape[1]
    out = np.empty((ar, bc))
    cuts = np.linspace(0, ar, threads + 1).astype(int)

    def work(lo, hi):
        if hi > lo:
            lib.matmul(_p(a[lo:hi]), hi - lo, ac, _p(b), bc, _p(out[lo:hi]))

    th = [threading.Thread(target=work, args=(cuts[t], cuts[t + 1])) for t in range(threads)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    return out


def systems(threads):
    lib = _orc()
    t0 = time.perf_counter()
    A = gaussian(lib, 1, M, P)
    B = gaussian(lib, 2, Q, N)
    Xs = gaussian(lib, 3, P, Q)
    X0 = gaussian(lib, 4, P, Q)
    A1 = gaussian(lib, 5, M, RANK)
    A2 = gaussian(lib, 6, RANK, P)
    Ard = matmul_mt(lib, A1, A2, threads)
    Ard *= 1.0 / np.sqrt(RANK)
    del A1, A2
    out = {}
    for name, a in (("full", A), ("rankdef", Ard)):
        T = matmul_mt(lib, a, Xs, threads)
        out[name] = (a, matmul_mt(lib, T, B, threads))
        del T
    print(f"[pin] inputs generated in {time.perf_counter() - t0:.1f}s", file=sys.stderr, flush=True)
    return out, B, Xs, X0


def probes():
    rng = np.random.default_rng(20251020)
    return rng.standard_normal((N_PROBES, P)), rng.standard_normal((N_PROBES, Q))


def digest(X, X0, r_sq):
    U, V = probes()
    return {"x_fro_sq": float(np.sum(X * X)), "dx_fro_sq": float(np.sum((X - X0) ** 2)),
            "x_rows": X[SAMPLE_ROWS].copy(), "x_probes": np.einsum("kp,pq,kq->k", U, X, V),
            "r_sq": np.asarray(r_sq, dtype=np.float64).copy()}


def ref_side(args):
    assert O.ref_available(), "oracle/_ref/libaxbref.so not built (make -C oracle)"
    sysd, B, Xs, X0 = systems(args.threads)
    lib = O.ref()
    res = {}

    def one(name, method, theta, sysname):
        A, Cm = sysd[sysname]
        cfg = O.make_config(method=method, theta=theta, stop_kind=O.SOLUTION_RRN, tol=0.0,
                            reference=Xs, seed=SOLVER_SEED, max_iter=10 ** 9, refresh_interval=1000)
        t0 = time.perf_counter()
        s = O.Solver(lib, A, B, Cm, X0, cfg)
        ctor = time.perf_counter() - t0
        t0 = time.perf_counter()
        rows = s.steps(args.steps)
        loop = time.perf_counter() - t0
        d = digest(s.X(), X0, s.r_sq())
        d.update(rows=rows.astype(np.int64), alpha=s.alpha, ctor_s=ctor, loop_s=loop)
        res[name] = d
        print(f"[pin] {name}: ctor {ctor:.1f}s, {args.steps} steps {loop:.1f}s "
              f"({1e3 * loop / args.steps:.1f} ms/step), alpha={d['alpha']:.17g}",
              file=sys.stderr, flush=True)
        del s

    th = [threading.Thread(target=one, args=v) for v in VARIANTS]
    for t in th:
        t.start()
    for t in th:
        t.join()
    flat = {"steps": np.int64(args.steps), "root_seed": np.int64(ROOT_SEED)}
    for name, d in res.items():
        for k, v in d.items():
            flat[f"{name}.{k}"] = np.asarray(v)
    np.savez_compressed(FIXTURE, **flat)
    print(f"[pin] wrote {FIXTURE}", file=sys.stderr)


def rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def compare(d, fx, name):
    return {"x_fro_sq": abs(d["x_fro_sq"] - float(fx[f"{name}.x_fro_sq"])) / float(fx[f"{name}.x_fro_sq"]),
            "dx_fro_sq": abs(d["dx_fro_sq"] - float(fx[f"{name}.dx_fro_sq"])) / float(fx[f"{name}.dx_fro_sq"]),
            "x_rows": rel(d["x_rows"], fx[f"{name}.x_rows"]),
            "x_probes": rel(d["x_probes"], fx[f"{name}.x_probes"]),
            "r_sq": rel(d["r_sq"], fx[f"{name}.r_sq"])}


def gpu_side(args):
    import paper_2408_05444_b200 as axb

    fx = np.load(FIXTURE)
    steps = int(fx["steps"])
    sysd, B, Xs, X0 = systems(args.threads)
    ok = True
    for name, method, theta, sysname in VARIANTS:
        if args.only and name not in args.only.split(","):
            continue
        A, Cm = sysd[sysname]
        alpha = float(fx[f"{name}.alpha"])
        meth = {O.GRBK: axb.Method.grbk(), O.MWRBK: axb.Method.mwrbk()}.get(method) or axb.Method.rgrbk(theta)
        rows_ref = fx[f"{name}.rows"].astype(np.int64)
        out = {"variant": name, "steps": steps, "alpha_ref": alpha}
        for mode in ("self", "replay"):
            cfg = axb.SolveConfig(method=meth, alpha_rule=axb.AlphaRule.Safe,
                                  stop=axb.StopRule.solution_rrn(0.0, Xs), max_iter=10 ** 9,
                                  seed=SOLVER_SEED, refresh_interval=1000)
            s = axb.Solver(A, B, Cm, X0, cfg, axb.Options(alpha_override=alpha, **args.opts))
            if mode == "self":
                rows = s.steps(steps).astype(np.int64)
                mism = np.nonzero(rows != rows_ref)[0]
                out["self_rows_identical"] = bool(mism.size == 0)
                out["self_first_mismatch"] = int(mism[0]) if mism.size else None
            else:
                s.replay(rows_ref.astype(np.uint64))
            d = digest(s.X(), X0, s.residual_row_sq())
            out[f"{mode}_rel"] = compare(d, fx, name)
            del s
        x_ok = all(v <= 1e-10 for k, v in out["replay_rel"].items() if k != "r_sq")
        r_ok = out["replay_rel"]["r_sq"] <= 1e-9
        out["pass"] = bool(out["self_rows_identical"] and x_ok and r_ok)
        ok &= out["pass"]
        print(json.dumps(out), flush=True)
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("side", choices=["ref", "gpu"])
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 8)
    ap.add_argument("--only", default="")
    ap.add_argument("--persist", type=int, default=None, help="Options.persist override (gpu side)")
    args = ap.parse_args()
    args.opts = {}
    if args.side == "ref":
        ref_side(args)
    else:
        sys.exit(0 if gpu_side(args) else 1)


if __name__ == "__main__":
    main()
