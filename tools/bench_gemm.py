"""K1 timing: the DMMA residual contraction against cuBLAS DGEMM (library, scale only).

  python tools/bench_gemm.py 3          # checkpoint (C − (A·X)·B + drift) at config 3
  python tools/bench_gemm.py pure       # pure GEMMs D = C − A·B at the config-3 / config-5 shapes

AXB_GEMM_TMA=0 selects the cp.async-fed kernel, the default is the TMA-fed one.
"""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import torch

import paper_2408_05444_b200 as axb
from paper_2408_05444_b200 import _lib


def pure():
    lib = _lib.load()
    for (M, N, K) in ((8192, 2048, 2048), (8192, 8192, 2048), (65536, 8192, 8192), (16384, 32768, 8192)):
        A = torch.randn(M, K, dtype=torch.float64, device="cuda")
        B = torch.randn(K, N, dtype=torch.float64, device="cuda")
        Cm = torch.randn(M, N, dtype=torch.float64, device="cuda")
        D = torch.empty_like(Cm)
        flops = 2.0 * M * N * K
        reps = 5 if flops < 1e13 else 2
        ms = C.c_double()
        torch.cuda.synchronize()
        rc = lib.axb_debug_dgemm(A.data_ptr(), B.data_ptr(), Cm.data_ptr(), D.data_ptr(), M, N, K, 0,
                                 reps, C.byref(ms))
        assert rc == 0, rc
        ref = Cm - A @ B
        err = (D - ref).norm().item() / ref.norm().item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            torch.addmm(Cm, A, B, beta=1.0, alpha=-1.0, out=D)
        e1.record()
        torch.cuda.synchronize()
        cb = e0.elapsed_time(e1) / reps
        print(f"D = C - A.B  {M}x{N}x{K}: K1 {ms.value:.3f} ms {flops / ms.value / 1e9:.2f} TFLOP/s | "
              f"cuBLAS {cb:.3f} ms {flops / cb / 1e9:.2f} TFLOP/s | rel diff {err:.1e}", flush=True)
        del A, B, Cm, D, ref
        torch.cuda.empty_cache()
    # Gram tile (b_trans): D = A·Aᵀ
    M, K = 8192, 2048
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    D = torch.empty(M, M, dtype=torch.float64, device="cuda")
    ms = C.c_double()
    rc = lib.axb_debug_dgemm(A.data_ptr(), A.data_ptr(), None, D.data_ptr(), M, M, K, 1, 3, C.byref(ms))
    assert rc == 0, rc
    ref = A @ A.T
    print(f"D = A.A^T {M}x{M}x{K}: K1 {ms.value:.3f} ms {2.0 * M * M * K / ms.value / 1e9:.2f} TFLOP/s | "
          f"rel diff {(D - ref).norm().item() / ref.norm().item():.1e}", flush=True)


def checkpoint(cfg_id):
    from bench import CONFIGS, make_inputs_device, solver_config

    cfg = CONFIGS[cfg_id]
    A, B, Cm, X0, Xs = make_inputs_device(cfg, 1000, 0)
    s = axb.Solver(A, B, Cm, X0, solver_config(axb, Xs, 10 ** 9), axb.Options(spectral_max_iter=200000))
    m, p, q, n = cfg["m"], cfg["p"], cfg["q"], cfg["n"]
    flops = 2 * m * p * q + 2 * m * q * n
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.checkpoint()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"checkpoint {dt * 1e3:.2f} ms  -> {flops / dt / 1e12:.2f} TFLOP/s (2mpq+2mqn = {flops:.3e})",
              flush=True)
    if cfg_id == 3:  # cuBLAS DGEMM pair for scale (library, tool-side only)
        Xd = torch.randn(p, q, dtype=torch.float64, device="cuda")
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            T = A @ Xd
            R = Cm - T @ B
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            print(f"cuBLAS DGEMM pair {dt * 1e3:.2f} ms -> {flops / dt / 1e12:.2f} TFLOP/s", flush=True)


if __name__ == "__main__":
    arg = sys.argv[1] if len(sys.argv) > 1 else "3"
    pure() if arg == "pure" else checkpoint(int(arg))
