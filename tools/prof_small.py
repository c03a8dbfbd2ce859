"""Config-1 GRBK on the persistent latency kernel: one warm batch, then one
2000-iteration batch (the launch `tools/prof_small.sh` captures with ncu)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle_lib as O
import paper_2408_05444_b200 as axb
orc = O.oracle()
A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)
cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X), seed=42,
                      refresh_interval=0)
s = axb.Solver(A, B, Cm, None, cfg)
s.steps(50)
s.steps(2000)
print(f"{s.last_timing()['loop_ms'] / 2000 * 1e3:.2f} us/iteration")
