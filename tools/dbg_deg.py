import os, sys, subprocess
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O
orc = O.oracle()
A, B, X, Cm = O.generate(orc, 17, 3, 2, 5, 7)
cfg_o = O.make_config(method=O.GRBK, stop_kind=O.SOLUTION_RRN, tol=0.0, reference=X, seed=6, max_iter=200000, refresh_interval=0)
so = O.Solver(orc, A, B, Cm, None, cfg_o)
print("oracle alpha", repr(so.alpha), "rows", so.steps(12))
code = r'''
import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, oracle_lib as O, paper_2408_05444_b200 as axb
orc = O.oracle()
A, B, X, Cm = O.generate(orc, 17, 3, 2, 5, 7)
cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X), max_iter=200000, seed=6, refresh_interval=0)
s = axb.Solver(A, B, Cm, None, cfg)
print("alpha", repr(s.alpha()), "rsq", s.residual_row_sq(), "rows", s.steps(12))
'''
for env in ({"AXB_PERSIST_LAT": "0"}, {"AXB_PERSIST_LAT": "256"}, {"AXB_PERSIST": "0"}):
    e = dict(os.environ); e.update(env)
    r = subprocess.run([sys.executable, "-c", code], env=e, capture_output=True, text=True)
    print(env, r.stdout.strip(), r.stderr.strip()[-300:])
