"""Time the DMMA residual contraction (checkpoint = C − (A·X)·B + drift) at config 3."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2408_05444_b200 as axb
from bench import CONFIGS, make_inputs_device, solver_config
cfg = CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 3]
A, B, C, X0, Xs = make_inputs_device(cfg, 1000, 0)
s = axb.Solver(A, B, C, X0, solver_config(axb, Xs, 10**9), axb.Options(spectral_max_iter=200000))
m, p, q, n = cfg["m"], cfg["p"], cfg["q"], cfg["n"]
flops = 2 * m * p * q + 2 * m * q * n
for rep in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s.checkpoint()
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"checkpoint {dt*1e3:.2f} ms  -> {flops/dt/1e12:.2f} TFLOP/s (2mpq+2mqn = {flops:.3e})")
# cuBLAS DGEMM for comparison (library, test-side only)
Ad = A.clone(); Xd = X0.clone(); Bd = B.clone()
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    T = Ad @ Xd; R = C - T @ Bd
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"cuBLAS DGEMM pair {dt*1e3:.2f} ms -> {flops/dt/1e12:.2f} TFLOP/s")
