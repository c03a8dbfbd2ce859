"""Time to ‖X−X*‖/‖X*‖ < 1e-6 on config 3 (A 8192×2048, B 2048×8192 N(0,1), X0 N(0,1)),
ME-GRBK through run() with the reference's default refresh every 1000 steps."""
import json, sys, time
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device, solver_config

cfg = CONFIGS[3]
A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
t0 = time.perf_counter()
s = axb.Solver(A, B, C, X0, solver_config(axb, Xs, 3 * 10 ** 6), axb.Options(spectral_max_iter=200000))
torch.cuda.synchronize()
setup = time.perf_counter() - t0
rep = s.run()
out = {"config": cfg["desc"], "method": "grbk", "stop": "||X-X*||_F/||X*||_F < 1e-6 (solution_rrn 1e-12)",
       "iterations": rep.iterations, "loop_seconds": round(rep.wall_seconds, 3),
       "setup_seconds": round(setup, 3), "final_rel_error": rep.final_rrn ** 0.5,
       "terminated_by": rep.terminated_by.name, "refresh_interval": 1000,
       "us_per_iteration": round(rep.wall_seconds / max(rep.iterations, 1) * 1e6, 2)}
print(json.dumps(out), flush=True)
