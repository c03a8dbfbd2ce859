"""Config 4 (one 1024×1024 blur channel): iterations/s, dense operands (the
latency body: BᵀB cached, zero-Gram rows skipped) against CSR operands (the
sparse path: only stored entries and the touched R rows move)."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

import configs  # noqa: E402
import paper_2408_05444_b200 as axb  # noqa: E402

for hb in (7, 15):
    A, B, Xs, Cm = configs.config4_channel(seed=4, nn=1024, half_band=hb)
    for label, a, b in (("dense", A, B), ("csr", sp.csr_matrix(A), sp.csr_matrix(B))):
        cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0), seed=1,
                              refresh_interval=1000, max_iter=10 ** 9)
        s = axb.Solver(a, b, Cm, None, cfg, axb.Options(spectral_max_iter=200000))
        s.steps(100)
        s.steps(5000)
        t = s.last_timing()
        rows = s.steps(200)
        print(f"half-band {hb} {label}: {5000 / (t['loop_ms'] / 1e3):.0f} it/s, "
              f"{t['loop_ms'] / 5000 * 1e3:.2f} us/it, alpha {s.alpha():.6e}, "
              f"rel residual {s.current_residual_rel():.3e}, rows[:4] {rows[:4].tolist()}", flush=True)
        del s
