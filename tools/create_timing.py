import sys, time, os
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
import paper_2408_05444_b200 as axb
orc = O.oracle()
A, B, X, Cm = O.generate(orc, 100, 500, 100, 80, 400)
cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-12, X), seed=1)
axb.Solver(A, B, Cm, None, cfg)
t0 = time.perf_counter(); hs = [axb.Solver(A, B, Cm, None, cfg) for _ in range(40)]; t1 = time.perf_counter()
reps = axb.run_many(hs); t2 = time.perf_counter()
print(f"LAT={os.environ.get('AXB_PERSIST_LAT','auto')}: create {1e3*(t1-t0)/40:.2f} ms/handle, run_many 40 solves {t2-t1:.3f} s, its {reps[0].iterations}")
