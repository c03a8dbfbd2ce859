import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, oracle_lib as O, paper_2408_05444_b200 as axb
orc = O.oracle()
for (m, p, q, n) in ((2000, 100, 80, 1000), (2048, 64, 32, 1400), (1600, 64, 32, 1400), (1900, 64, 32, 400)):
    A, B, X, Cm = O.generate(orc, 3, m, p, q, n)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X), seed=1, refresh_interval=0)
    try:
        s = axb.Solver(A, B, Cm, None, cfg); s.steps(100); print(m, p, q, n, "ok", s.last_timing()["loop_ms"])
    except Exception as e:
        print(m, p, q, n, "FAIL", e)
