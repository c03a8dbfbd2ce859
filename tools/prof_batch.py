"""One run_many batch of config-1 solves (for ncu on k_persist_batch)."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
import paper_2408_05444_b200 as axb
orc = O.oracle()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 148
A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)
hs = [axb.Solver(A, B, Cm, None, axb.SolveConfig(method=axb.Method.grbk(),
                 stop=axb.StopRule.solution_rrn(1e-12, X), seed=t, max_iter=2000)) for t in range(n)]
t0 = time.perf_counter()
reps = axb.run_many(hs)
dt = time.perf_counter() - t0
its = sum(r.iterations for r in reps)
print(f"{n} solves x {reps[0].iterations} its: {dt:.3f} s, {its / dt:.0f} it/s, {dt / reps[0].iterations * 1e6:.1f} us per batched iteration")
