"""Config 5 at full size (A 65536×8192, B 8192×32768): the row-sharded path gives the
single-GPU index sequence and X ("index sequence and X must be identical
(≤1e-10) across 1/2/4/8 GPUs").

One B200: the unsharded solver first, then the sharded solver over a real 1-rank NCCL
communicator, then world = 2, 4, 8 with every rank a host thread and its own handle on
this device through the library's in-process collective emulation (no rank's kernel
waits on another's).  Each rank gets its contiguous rows of the same global A and C
(bench.py's generator), full B and X*; budget K steps, so G is not cached (g = A·A_iᵀ
per step on every path).

    python tools/config5_shard_invariance.py [--steps 300] [--worlds 1,2,4,8]
"""
import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_05444_b200 as axb  # noqa: E402
from paper_2408_05444_b200 import shard  # noqa: E402
from bench import CONFIGS, make_inputs_device, solver_config  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    K = args.steps
    cfg = CONFIGS[5]
    A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
    opts = dict(spectral_max_iter=200000)

    t0 = time.perf_counter()
    s = axb.Solver(A, B, C, X0, solver_config(axb, Xs, K), axb.Options(**opts))
    setup = time.perf_counter() - t0
    rows1 = s.steps(K)
    X1 = s.X()
    alpha1 = s.alpha()
    print(json.dumps({"run": "single GPU (unsharded)", "steps": K, "setup_s": round(setup, 2),
                      "loop_ms": round(s.last_timing()["loop_ms"], 2), "alpha": alpha1,
                      "gram_cached": bool(s.gram_cached())}), flush=True)
    del s
    torch.cuda.empty_cache()

    bad = False
    for world in [int(w) for w in args.worlds.split(",")]:
        ml = cfg["m"] // world
        if world == 1:
            comms = [shard.nccl_comm_create(1, shard.nccl_unique_id(), 0, 0)]
            kind = "sharded path, real 1-rank NCCL communicator"
        else:
            comms = shard.emulated_comms(world)
            kind = f"sharded path, {world} ranks emulated on one device"
        out = [None] * world
        errs = []

        def rank(r):
            try:
                sl = slice(r * ml, (r + 1) * ml)
                sr = shard.sharded_solver(A[sl], B, C[sl], X0, solver_config(axb, Xs, K), comms[r],
                                          world, r, device=0, **opts)
                rows = sr.steps(K)
                ms = sr.last_timing()["loop_ms"]
                Xr = sr.X()  # every rank calls it (it may gather X's row slices)
                out[r] = (rows, Xr if r == 0 else None, sr.alpha(), ms)
                del sr
            except Exception as e:  # noqa: BLE001
                errs.append(repr(e))

        t0 = time.perf_counter()
        th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=1200)
        wall = time.perf_counter() - t0
        for c in comms:
            shard.nccl_comm_destroy(c)
        torch.cuda.empty_cache()
        if errs or any(o is None for o in out):
            print(json.dumps({"run": kind, "error": errs[:2]}), flush=True)
            bad = True
            continue
        mism = [int(np.count_nonzero(o[0] != rows1)) for o in out]
        first = [int(np.nonzero(o[0] != rows1)[0][0]) if m else None for o, m in zip(out, mism)]
        line = {"run": kind, "world": world, "steps": K, "index_mismatches_per_rank": mism,
                "first_mismatch_per_rank": first,
                "alpha_identical": all(o[2] == alpha1 for o in out),
                "X_rel_diff_vs_single_gpu": rel(out[0][1], X1),
                "rank0_loop_ms": round(out[0][3], 2), "wall_s": round(wall, 2)}
        print(json.dumps(line), flush=True)
        bad |= any(mism) or line["X_rel_diff_vs_single_gpu"] > 1e-10
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
