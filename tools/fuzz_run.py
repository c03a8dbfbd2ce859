"""Randomised run()-to-tolerance comparison (stop rule, refresh checkpoints,
confirm logic) against the oracle; plus the same systems batched through
run_many.  usage: python tools/fuzz_run.py [cases] [seed]"""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O
import paper_2408_05444_b200 as axb

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
orc = O.oracle()
meths = [(O.GRBK, None, lambda: axb.Method.grbk()), (O.MWRBK, None, lambda: axb.Method.mwrbk()),
         (O.RBK, None, lambda: axb.Method.rbk()), (O.RGRBK, 0.4, lambda: axb.Method.rgrbk(0.4))]
bad = 0
t0 = time.perf_counter()
handles, expect = [], []
for c in range(cases):
    p, q = int(rng.integers(2, 40)), int(rng.integers(2, 40))
    m, n = int(rng.integers(2 * p, 8 * p + 10)), int(rng.integers(2 * q, 8 * q + 10))
    tag, theta, meth = meths[rng.integers(0, len(meths))]
    A, B, X, Cm = O.generate(orc, int(rng.integers(1, 10 ** 6)), m, p, q, n)
    ri = int(rng.choice([0, 100, 1000]))
    so = O.Solver(orc, A, B, Cm, None, O.make_config(method=tag, theta=theta, seed=3,
                  stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=X, refresh_interval=ri, max_iter=60000))
    ro = so.run()[0]
    mk = lambda: axb.SolveConfig(method=meth(), stop=axb.StopRule.solution_rrn(1e-12, X), seed=3,  # noqa: E731
                                 refresh_interval=ri, max_iter=60000)
    rg = axb.Solver(A, B, Cm, None, mk()).run()
    handles.append(axb.Solver(A, B, Cm, None, mk()))
    it_o = int(ro.iterations)
    tb_o = int(ro.terminated_by)
    expect.append(it_o)
    ok = abs(rg.iterations - it_o) <= 2
    bad += 0 if ok else 1
    print(f"{'ok ' if ok else 'BAD'} case {c}: {m}x{p}.{q}x{n} {meth()} refresh {ri}: iterations "
          f"{rg.iterations} vs oracle {it_o} ({rg.terminated_by.name} / {tb_o}), final rrn {rg.final_rrn:.3e}",
          flush=True)
reps = axb.run_many(handles)
bb = sum(abs(r.iterations - e) > 2 for r, e in zip(reps, expect))
print(f"run(): {cases - bad}/{cases} within ±2 iterations; run_many batch: {cases - bb}/{cases}; "
      f"{time.perf_counter() - t0:.0f} s")
