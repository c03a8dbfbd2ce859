"""Replays ONE case of tools/fuzz_shard.py (same RNG walk) with diagnostics: the
first step where the sharded rows leave the oracle's, the oracle's ‖R‖/‖C‖ there,
whether the single-GPU path leaves at the same step, and how far the reference's
running ‖R‖² has drifted from the fresh sum of its own row norms by then.

    python tools/fuzz_shard_case.py <seed> <case>
"""
import sys, threading
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import shard

seed, case = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(seed)
orc = O.oracle()
meths = [(O.GRBK, None, lambda: axb.Method.grbk()), (O.MWRBK, None, lambda: axb.Method.mwrbk()),
         (O.RBK, None, lambda: axb.Method.rbk()), (O.BK, None, lambda: axb.Method.bk()),
         (O.RGRBK, 0.6, lambda: axb.Method.rgrbk(0.6))]
for c in range(case + 1):
    world = int(rng.choice([2, 4, 8]))
    ml = int(rng.integers(1, 900))
    m, p, q, n = ml * world, int(rng.integers(1, 120)), int(rng.integers(1, 90)), int(rng.integers(2, 3000))
    tag, theta, meth = meths[rng.integers(0, len(meths))]
    gram = int(rng.integers(0, 2))
    gseed = int(rng.integers(1, 10 ** 6))
steps = 120
print(f"case {case}: world {world} {m}x{p}.{q}x{n} {meth()} cache_gram={gram}")
A, B, X, Cm = O.generate(orc, gseed, m, p, q, n)
so = O.Solver(orc, A, B, Cm, None, O.make_config(method=tag, theta=theta, seed=9, stop_kind=O.SOLUTION_RRN,
              tol=0.0, reference=X, refresh_interval=0))
ro, rel, drift = [], [], []
cn = np.linalg.norm(Cm)
for k in range(steps):
    ro.append(int(so.steps(1)[0]))
    run = so.residual_fro_sq
    fresh = float(np.sum(so.r_sq()))
    rel.append(np.sqrt(max(run, 0)) / cn)
    drift.append(abs(run - fresh) / max(fresh, 1e-300))
ro = np.array(ro)
mk = lambda: axb.SolveConfig(method=meth(), stop=axb.StopRule.solution_rrn(0.0, X), seed=9, refresh_interval=0)
s1 = axb.Solver(A, B, Cm, None, mk(), axb.Options(cache_gram=gram))
r1 = s1.steps(steps)
m1 = np.nonzero(r1 != ro)[0]
print("single GPU first mismatch:", m1[:3])
comms = shard.emulated_comms(world)
out = [None] * world


def body(r):
    s = shard.sharded_solver(np.ascontiguousarray(A[r * ml:(r + 1) * ml]), B,
                             np.ascontiguousarray(Cm[r * ml:(r + 1) * ml]), None, mk(), comms[r], world, r,
                             cache_gram=gram)
    out[r] = s.steps(steps)


th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
[t.start() for t in th]
[t.join() for t in th]
mm = np.nonzero(out[0] != ro)[0]
print("sharded first mismatch:", mm[:3], "all ranks agree:", all(np.array_equal(out[0], o) for o in out))
for name, mmx, rows in (("single", m1, r1), ("sharded", mm, out[0])):
    if mmx.size:
        k = int(mmx[0])
        before = f"{rel[k - 1]:.3e}" if k else "(initial residual)"
        print(f"{name}: step {k}: oracle row {ro[k]}, device row {rows[k]}; oracle ||R||/||C|| after step {k - 1}: "
              f"{before}; reference running-vs-fresh ||R||^2 drift there: "
              f"{drift[k - 1] if k else 0:.3e}; ||R||/||C|| at step 0: {rel[0]:.3e}")
if p == 1:
    # A is one column: R0 = a·(x*B), so every row's ratio ‖R_l‖²/‖A_l‖² is the same
    # number in exact arithmetic and every greedy membership test is an exact tie
    ratios = so.r_sq() / np.maximum(so.a_sq(), 1e-300)
    print(f"p = 1: all {m} ratios ||R_l||^2/||A_l||^2 tie to rounding (spread "
          f"{(ratios.max() - ratios.min()) / ratios.max():.2e}): the last bit of a row norm decides")
