"""Setup-time breakdown of Solver(...) at config 3 (host pinned and device inputs)."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device, solver_config
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
host = {}
for k, t in (("A", A), ("B", B), ("C", C), ("X0", X0), ("Xs", Xs)):
    if t is None: host[k] = None; continue
    h = torch.empty(t.shape, dtype=torch.float64, pin_memory=True); h.copy_(t); host[k] = h.numpy()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = axb.Solver(A, B, C, X0, solver_config(axb, Xs, 10**9), axb.Options(spectral_max_iter=200000))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    s2 = axb.Solver(host["A"], host["B"], host["C"], host["X0"], solver_config(axb, host["Xs"], 10**9),
                    axb.Options(spectral_max_iter=200000))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"device-input setup {1e3*(t1-t0):.1f} ms, pinned-host setup {1e3*(t2-t1):.1f} ms, alpha {s.alpha():.10e} {s2.alpha():.10e}")
    del s, s2
