"""Config 4 (one 1024×1024 blur channel): iterations/s with the zero-Gram-row skip."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import paper_2408_05444_b200 as axb
import configs
for hb in (7, 15):
    A, B, Xs, Cm = configs.config4_channel(seed=4, nn=1024, half_band=hb)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0), seed=1,
                          refresh_interval=1000)
    s = axb.Solver(A, B, Cm, None, cfg, axb.Options(spectral_max_iter=200000))
    s.steps(100)
    s.steps(2000)
    t = s.last_timing()
    print(f"half-band {hb}: {2000 / (t['loop_ms'] / 1e3):.0f} it/s, {t['loop_ms'] / 2000 * 1e3:.1f} us/it,"
          f" alpha {s.alpha():.6e}, rel residual {s.current_residual_rel():.3e}")
