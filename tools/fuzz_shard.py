"""Randomised shapes on the row-sharded path (world 2/4/8 emulated on one GPU,
ranks as host threads) against the oracle.
usage: python tools/fuzz_shard.py [cases] [seed] [only: comma-separated case numbers]
A case that leaves the oracle's rows is followed by a diagnosis line (tools/fuzz_diag.py)."""
import sys, threading, time
sys.path.insert(0, "."); sys.path.insert(0, "tests"); sys.path.insert(0, "tools")
import numpy as np
import oracle_lib as O
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import shard
from fuzz_diag import diagnose

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
only = {int(x) for x in sys.argv[3].split(",")} if len(sys.argv) > 3 else None
orc = O.oracle()
meths = [(O.GRBK, None, lambda: axb.Method.grbk()), (O.MWRBK, None, lambda: axb.Method.mwrbk()),
         (O.RBK, None, lambda: axb.Method.rbk()), (O.BK, None, lambda: axb.Method.bk()),
         (O.RGRBK, 0.6, lambda: axb.Method.rgrbk(0.6))]
bad = 0
t0 = time.perf_counter()
for c in range(cases):
    world = int(rng.choice([2, 4, 8]))
    ml = int(rng.integers(1, 900))
    m, p, q, n = ml * world, int(rng.integers(1, 120)), int(rng.integers(1, 90)), int(rng.integers(2, 3000))
    tag, theta, meth = meths[rng.integers(0, len(meths))]
    gram = int(rng.integers(0, 2))
    steps = 120
    gseed = int(rng.integers(1, 10 ** 6))
    if only is not None and c not in only:
        continue
    A, B, X, Cm = O.generate(orc, gseed, m, p, q, n)
    desc = f"case {c}: world {world} {m}x{p}.{q}x{n} {meth()} cache_gram={gram}"
    try:
        so = O.Solver(orc, A, B, Cm, None, O.make_config(method=tag, theta=theta, seed=9,
                      stop_kind=O.SOLUTION_RRN, tol=0.0, reference=X, refresh_interval=0))
        ro = so.steps(steps)
        Xo = so.X()
        comms = shard.emulated_comms(world)
        out, errs = [None] * world, []

        def body(r):
            try:
                cfg = axb.SolveConfig(method=meth(), stop=axb.StopRule.solution_rrn(0.0, X), seed=9,
                                      refresh_interval=0)
                s = shard.sharded_solver(np.ascontiguousarray(A[r * ml:(r + 1) * ml]), B,
                                         np.ascontiguousarray(Cm[r * ml:(r + 1) * ml]), None, cfg,
                                         comms[r], world, r, cache_gram=gram)
                out[r] = (s.steps(steps), s.X())
            except Exception as e:  # noqa: BLE001
                errs.append(e)

        th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=300)
        for cm in comms:
            shard.nccl_comm_destroy(cm)
        if errs:
            raise errs[0]
        worst = 0
        ok = True
        first = None
        for rows, Xr in out:
            mism = np.nonzero(rows != ro)[0]
            if mism.size and first is None:
                first = int(mism[0])
            e = np.linalg.norm(Xr - Xo) / max(np.linalg.norm(Xo), 1e-300)
            worst = max(worst, e)
            ok &= mism.size == 0 and e <= 1e-10
        if not ok:
            bad += 1
        print(f"{'ok ' if ok else 'BAD'} {desc}: |dX|/|X| {worst:.2e}", flush=True)
        if first is not None:
            print("    " + diagnose(orc, A, B, Cm, X, tag, theta, 9, first), flush=True)
    except Exception as ex:  # noqa: BLE001
        bad += 1
        print(f"ERR {desc}: {type(ex).__name__}: {ex}", flush=True)
print(f"{cases - bad}/{cases} ok in {time.perf_counter() - t0:.0f} s")
