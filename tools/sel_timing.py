import ctypes as C, sys
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import _lib
from bench import CONFIGS, make_inputs_device
lib = _lib.load(); lib.axb_solver_debug_state.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
cfg = CONFIGS[int(sys.argv[1])]
A, B, Cm, X0, Xs = make_inputs_device(cfg, 1000, 0)
sc = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-12, Xs), seed=42, refresh_interval=0)
s = axb.Solver(A, B, Cm, X0, sc, axb.Options(spectral_max_iter=200000))
for it in range(4):
    s.steps(5)
    d = (C.c_uint64 * 8)(); lib.axb_solver_debug_state(s._h, d)
    print("reduce->sel", (d[0]-d[7])/1e3, "groups", (d[1]-d[0])/1e3, "prefix", (d[2]-d[1])/1e3, "search", (d[3]-d[2])/1e3, "fallback", (d[4]-d[3])/1e3, "us; selections", d[5], "fallbacks", d[6])
