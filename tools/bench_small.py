"""Per-iteration latency on small systems: persistent kernel vs graph path."""
import os, sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np
import oracle_lib as O, configs
import paper_2408_05444_b200 as axb
orc = O.oracle()
cases = {"config1": O.generate(orc, 7, 500, 100, 80, 400)[:4]}
A2, B2, X2, C2 = configs.config2(seed=2); cases["config2"] = (A2, B2, X2, C2)
A4, B4, X4, C4 = configs.config4_channel(seed=4, nn=1024, half_band=7); cases["config4"] = (A4, B4, X4, C4)
for name, (A, B, X, Cm) in cases.items():
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X), seed=42,
                          refresh_interval=0)
    s = axb.Solver(A, B, Cm, None, cfg, axb.Options(spectral_max_iter=200000))
    s.steps(50); s.steps(3000)
    print(f"{name} [persist={os.environ.get('AXB_PERSIST', 'auto')} grid={os.environ.get('AXB_PERSIST_GRID', 'sms')}]: {s.last_timing()['loop_ms'] / 3000 * 1e3:.2f} us/iteration")

# run() to tolerance on config 1 (the bench's time_to_tol workload)
A, B, X, Cm = cases["config1"]
cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-12, X), seed=42,
                      refresh_interval=1000)
s = axb.Solver(A, B, Cm, None, cfg)
rep = s.run()
print(f"config1 run() [persist={os.environ.get('AXB_PERSIST', 'auto')}]: {rep.iterations} its in"
      f" {rep.wall_seconds:.4f} s = {rep.wall_seconds / rep.iterations * 1e6:.2f} us/iteration")
