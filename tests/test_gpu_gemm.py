"""K1 (DMMA GEMM) — the TMA-fed kernel against the cp.async one and numpy.

Both kernels accumulate every output element over k in the same order (DMMA
k-steps of 4, ascending), so the residual R0 = C − (A·X0)·B and the cached Gram
G = A·Aᵀ must agree BITWISE between them; numpy (a different summation order)
agrees to rounding.  Shapes cover partial tiles in M, N and K, and operands whose
pitch is odd (no 16-byte alignment: the cp.async kernel is the only path).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    (64, 16, 16, 128),      # exactly one tile
    (130, 50, 34, 150),     # partial tiles everywhere
    (500, 100, 80, 400),    # config 1
    (257, 36, 130, 1026),   # several k tiles, ragged N
    (96, 24, 18, 272),      # K = 18: partial last k tile (zero-filled by the map)
    (70, 7, 9, 33),         # odd pitches: falls back to the cp.async kernel
]


def _residual(axb, A, B, C, X0, tma, cache_gram=-1, steps=0):
    os.environ["AXB_GEMM_TMA"] = "1" if tma else "0"
    try:
        cfg = axb.SolveConfig(method=axb.Method.mwrbk(), max_iter=10 ** 6, refresh_interval=0)
        s = axb.Solver(A, B, C, X0, cfg, axb.Options(cache_gram=cache_gram))
        rows = s.steps(steps) if steps else None
        return s.R(), s.X(), rows, s.exact_residual_rel()
    finally:
        os.environ.pop("AXB_GEMM_TMA", None)


@pytest.mark.parametrize("shape", SHAPES)
def test_r0_tma_equals_cp_async_bitwise(axb, shape):
    m, p, q, n = shape
    rng = np.random.default_rng(sum(shape))
    A, B = rng.standard_normal((m, p)), rng.standard_normal((q, n))
    X0, C = rng.standard_normal((p, q)), rng.standard_normal((m, n))
    R1, _, _, e1 = _residual(axb, A, B, C, X0, True)
    R0, _, _, e0 = _residual(axb, A, B, C, X0, False)
    assert np.array_equal(R1, R0), "TMA-fed and cp.async-fed DMMA kernels differ"
    assert e1 == e0
    Rn = C - (A @ X0) @ B
    assert np.linalg.norm(R1 - Rn) <= 1e-13 * np.linalg.norm(Rn)


@pytest.mark.parametrize("shape", [(130, 50, 34, 150), (300, 64, 48, 256)])
def test_gram_tma_equals_cp_async(axb, shape):
    """G = A·Aᵀ through the b_trans tile (k-contiguous boxes for both operands)."""
    m, p, q, n = shape
    rng = np.random.default_rng(7 + sum(shape))
    A, B = rng.standard_normal((m, p)), rng.standard_normal((q, n))
    Xs = rng.standard_normal((p, q))
    C = (A @ Xs) @ B
    _, X1, rows1, _ = _residual(axb, A, B, C, None, True, cache_gram=1, steps=60)
    _, X0, rows0, _ = _residual(axb, A, B, C, None, False, cache_gram=1, steps=60)
    assert np.array_equal(rows1, rows0)
    assert np.array_equal(X1, X0)
    # and against g = A·A_iᵀ formed per step (no cached Gram at all)
    _, Xg, rowsg, _ = _residual(axb, A, B, C, None, True, cache_gram=0, steps=60)
    assert np.array_equal(rows1, rowsg)
    assert np.linalg.norm(X1 - Xg) <= 1e-12 * np.linalg.norm(Xg)


def test_residual_chain_order(axb):
    """R0 = C − A·X0·B with the product associated as A·(X0·B) (taken when it is
    ≥ 5% cheaper, e.g. config 5) and as the reference's (A·X0)·B: same product to
    rounding, both within 1e-13 of numpy."""
    m, p, q, n = 512, 64, 64, 256  # pn(q+m) = 0.90·mq(p+n): the auto rule picks A·(X·B)
    rng = np.random.default_rng(99)
    A, B = rng.standard_normal((m, p)), rng.standard_normal((q, n))
    X0, C = rng.standard_normal((p, q)), rng.standard_normal((m, n))
    Rn = C - (A @ X0) @ B
    out = {}
    for mode in ("0", "1", None):
        if mode is None:
            os.environ.pop("AXB_CHAIN_XB", None)
        else:
            os.environ["AXB_CHAIN_XB"] = mode
        try:
            out[mode], _, _, _ = _residual(axb, A, B, C, X0, True)
        finally:
            os.environ.pop("AXB_CHAIN_XB", None)
        assert np.linalg.norm(out[mode] - Rn) <= 1e-13 * np.linalg.norm(Rn)
    assert np.array_equal(out[None], out["1"]), "the auto rule should pick A·(X·B) here"
    assert np.linalg.norm(out["0"] - out["1"]) <= 1e-14 * np.linalg.norm(Rn)


@pytest.mark.parametrize("b_trans", [0, 1])
def test_debug_dgemm_export(axb, b_trans):
    """axb_debug_dgemm (K1 timed alone, device pointers): D = C − A·B and D = A·Bᵀ."""
    import ctypes as C

    import torch

    from paper_2408_05444_b200 import _lib

    lib = _lib.load()
    M, N, K = 200, 144, 96
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(M, K, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((N, K) if b_trans else (K, N), dtype=torch.float64, device="cuda", generator=g)
    Cm = torch.randn(M, N, dtype=torch.float64, device="cuda", generator=g)
    D = torch.empty_like(Cm)
    ms = C.c_double()
    torch.cuda.synchronize()
    rc = lib.axb_debug_dgemm(A.data_ptr(), B.data_ptr(), None if b_trans else Cm.data_ptr(), D.data_ptr(),
                             M, N, K, b_trans, 2, C.byref(ms))
    assert rc == 0 and ms.value > 0.0
    ref = A @ B.T if b_trans else Cm - A @ B
    assert (D - ref).norm().item() <= 1e-13 * ref.norm().item()
    assert lib.axb_debug_timeline(None, 0) in (0, 1)  # 1 only in a -DAXB_TRACE_TIMELINE build
