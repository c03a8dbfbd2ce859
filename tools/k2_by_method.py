"""K2 in-pipeline time at config 5 by selection method (isolates the last-CTA selection tail)."""
import sys
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device
cfg = CONFIGS[5]
A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
for name, meth in (("mwrbk", axb.Method.mwrbk()), ("grbk", axb.Method.grbk()), ("rbk", axb.Method.rbk())):
    sc = axb.SolveConfig(method=meth, stop=axb.StopRule.solution_rrn(1e-12, Xs), seed=42, refresh_interval=0)
    s = axb.Solver(A, B, C, X0, sc, axb.Options(spectral_max_iter=200000))
    s.steps(3)
    s.set_profiling(True)
    s.steps(20)
    print(name, s.kernel_times())
    s.set_profiling(False)
    del s
    torch.cuda.empty_cache()
