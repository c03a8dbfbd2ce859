"""GPU: CSR operands kept sparse on the device.

The reference runs Solver<SparseMatrix, BMat> over stored entries only: the CSR
Gram (matrix.hpp:496-535), y = B·R_iᵀ over B's stored entries (solver.hpp:489-492),
the X update over nz(A_i) (:272-273) and the R update over nz(G_i) (:294-295).
The device keeps A, G = A·Aᵀ and B in CSR (A is never expanded) and its
persistent body iterates the same entries.  Adding the exact zeros of a dense
form changes no reference value, so the dense oracle is the sparse reference
bit for bit (checked here against oracle/_ref's Solver<SparseMatrix,…> too);
bar: the oracle's rows, X within 1e-10 (test_solver.cpp:546-561 pattern).
"""
import numpy as np
import pytest
import scipy.sparse as sp

import configs
import oracle_lib as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def method(axb, tag, theta=None):
    return {O.BK: axb.Method.bk(), O.RBK: axb.Method.rbk(), O.GRBK: axb.Method.grbk(),
            O.RGRBK: axb.Method.rgrbk(theta if theta is not None else 0.5),
            O.MWRBK: axb.Method.mwrbk()}[tag]


def banded(rng, rows, cols, hb):
    M = np.zeros((rows, cols))
    for i in range(rows):
        c = int(i * cols / rows)
        for j in range(max(0, c - hb), min(cols, c + hb + 1)):
            M[i, j] = np.exp(-0.2 * (j - c) ** 2) + 0.05 * rng.standard_normal()
    return M


@pytest.mark.parametrize("tag,theta", [(O.GRBK, None), (O.RGRBK, 0.3), (O.MWRBK, None),
                                       (O.RBK, None), (O.BK, None)])
@pytest.mark.parametrize("which", ["A", "B", "AB"])
@pytest.mark.parametrize("body", ["latency", "general"])
def test_csr_operands_match_oracle(axb, orc, tag, theta, which, body, monkeypatch):
    """Both persistent bodies: the latency body (m ≤ 2048; z = BᵀB·R_iᵀ over the
    CSR BᵀB) and the general body (z = yᵀB over Bᵀ's rows)."""
    if body == "general":
        monkeypatch.setenv("AXB_PERSIST_LAT", "0")
    rng = np.random.default_rng(11)
    m, p, q, n = 300, 240, 40, 160
    Ad, Bd = banded(rng, m, p, 4), banded(rng, q, n, 6)
    Xs = rng.standard_normal((p, q))
    Cm = (Ad @ Xs) @ Bd
    k = 800
    cfg_o = O.make_config(method=tag, theta=theta, seed=21, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=Xs, refresh_interval=0)
    so = O.Solver(orc, Ad, Bd, Cm, None, cfg_o)
    ro = so.steps(k)
    A = sp.csr_matrix(Ad) if "A" in which else Ad
    B = sp.csr_matrix(Bd) if "B" in which else Bd
    cfg = axb.SolveConfig(method=method(axb, tag, theta), stop=axb.StopRule.solution_rrn(0.0, Xs),
                          seed=21, refresh_interval=0)
    s = axb.Solver(A, B, Cm, None, cfg)
    assert s.alpha() == so.alpha
    rows = s.steps(k)
    mism = np.nonzero(rows.astype(np.int64) != ro.astype(np.int64))[0]
    assert mism.size == 0, f"first row mismatch at step {mism[:5]}"
    assert rel(s.X(), so.X()) <= 1e-10
    assert rel(s.residual_row_sq(), so.r_sq()) <= 1e-9
    # the incremental ‖X−X*‖² tracker (CSR A) against the exact metric
    assert s.current_metric() == pytest.approx(so.exact_metric(), rel=1e-8)
    if O.ref_available() and "A" in which:
        rr, Xr, _, al = O.ref().sparse_steps(sp.csr_matrix(Ad), B if "B" in which else Bd, Cm,
                                             None, cfg_o, k)
        np.testing.assert_array_equal(rr, ro)  # the sparse reference engine, bit for bit
        np.testing.assert_array_equal(Xr, so.X())
        assert al == so.alpha


def test_csr_x0_update_row_checkpoint_run(axb, orc):
    """X0 ≠ 0 (R0 = C − (A·X0)·B with the sparse product), update_row, a
    checkpoint (exact residual over CSR A) and run() with the refresh schedule."""
    rng = np.random.default_rng(5)
    m, p, q, n = 200, 160, 24, 96
    Ad, Bd = banded(rng, m, p, 3), rng.standard_normal((q, n))
    Xs, X0 = rng.standard_normal((p, q)), rng.standard_normal((p, q))
    Cm = (Ad @ Xs) @ Bd
    cfg_o = O.make_config(method=O.GRBK, seed=4, stop_kind=O.SOLUTION_RRN, tol=0.0, reference=Xs,
                          refresh_interval=0)
    so = O.Solver(orc, Ad, Bd, Cm, X0, cfg_o)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, Xs), seed=4,
                          refresh_interval=0)
    s = axb.Solver(sp.csr_matrix(Ad), Bd, Cm, X0, cfg)
    assert rel(s.R(), so.R()) <= 1e-13
    so.update_row(17)
    s.update_row(17)
    assert s.iteration() == so.iteration == 0
    assert rel(s.X(), so.X()) <= 1e-12
    np.testing.assert_array_equal(s.steps(300), so.steps(300))
    so.checkpoint()
    s.checkpoint()
    assert rel(s.R(), so.R()) <= 1e-10
    np.testing.assert_array_equal(s.steps(200), so.steps(200))
    assert s.exact_metric() == pytest.approx(so.exact_metric(), rel=1e-9)
    # run() to tolerance with refresh checkpoints on a well-conditioned banded A
    # (±2 iterations: the device's fresh ‖R‖² against the reference's running sum)
    for i in range(m):
        Ad[i, int(i * p / m)] += 2.0
    Cm = (Ad @ Xs) @ Bd
    cfg_o = O.make_config(method=O.MWRBK, stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=Xs,
                          refresh_interval=500, max_iter=200000)
    rep_o = O.Solver(orc, Ad, Bd, Cm, None, cfg_o).run()[0]
    assert rep_o.terminated_by == 0
    cfg = axb.SolveConfig(method=axb.Method.mwrbk(), stop=axb.StopRule.solution_rrn(1e-12, Xs),
                          refresh_interval=500, max_iter=200000)
    rep = axb.Solver(sp.csr_matrix(Ad), sp.csr_matrix(Bd), Cm, None, cfg).run()
    assert rep.terminated_by == axb.Terminated.Tolerance
    assert abs(rep.iterations - rep_o.iterations) <= 2


def test_restoration_shape_on_device(axb):
    """The reference's §6 restoration shape (imaging.hpp:183-196): a 256×256×3
    image, A the mn×mn CSR blur operator (build_blur_operator, 5×5 Gaussian,
    σ = 6, zero boundary), B = A_cᵀ (the paper's 3×3 mixing), observed
    C = A·X·A_cᵀ.  A dense A would be 34 GB; the device keeps it in CSR.  2000
    GRBK steps give the sparse reference engine's rows (oracle/_ref,
    Solver<SparseMatrix, DenseMatrix>) and X within 1e-10."""
    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    r = O.ref()
    A, Xs, Ac = r.blur_model(256, 256, 5, 6.0)
    B = np.ascontiguousarray(Ac.T)
    Cm = np.ascontiguousarray((A @ Xs) @ B)
    k = 2000
    cfg_o = O.make_config(method=O.GRBK, stop_kind=O.RESIDUAL_REL, tol=0.0, seed=8,
                          refresh_interval=0)
    rows_r, X_r, rs_r, al = r.sparse_steps(A, B, Cm, None, cfg_o, k)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0), seed=8,
                          refresh_interval=0)
    s = axb.Solver(A, B, Cm, None, cfg)
    assert s.alpha() == al
    rows = s.steps(k)
    mism = np.nonzero(rows.astype(np.int64) != rows_r.astype(np.int64))[0]
    assert mism.size == 0, f"first row mismatch at step {mism[:5]}"
    assert rel(s.X(), X_r) <= 1e-10
    assert rel(s.residual_row_sq(), rs_r) <= 1e-9


def test_config4_channel_csr(axb, orc):
    """A config-4 channel (1024², half-band 7) with banded CSR A = B: the
    restated engine's rows over 1500 GRBK steps, X within 1e-10, α bit for bit.
    (The reference constructor's power-iteration cap throws at n = 1024, SURVEY
    §0, so the oracle gets the reference's power iteration with a raised cap.)"""
    import ctypes as C

    A, B, Xs, Cm = configs.config4_channel(seed=4, nn=1024, half_band=7)
    st = C.c_int()
    spec = orc.spectral_norm(O._ptr(np.ascontiguousarray(B)), 1024, 1024, 1e-10, 200000,
                             C.byref(st), None)
    assert st.value == 0
    cfg_o = O.make_config(method=O.GRBK, seed=3, stop_kind=O.RESIDUAL_REL, tol=0.0,
                          refresh_interval=0, max_iter=10 ** 9)
    so = O.PreparedSolver(orc, A, B, Cm, np.zeros_like(Xs), Cm, A @ A.T, B.T @ B,
                          1.0 / (spec * spec), cfg_o)
    ro = so.steps(1500)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.residual_rel(0.0), seed=3,
                          refresh_interval=0, max_iter=10 ** 9)
    s = axb.Solver(sp.csr_matrix(A), sp.csr_matrix(B), Cm, None, cfg,
                   axb.Options(spectral_max_iter=200000))
    assert s.alpha() == 1.0 / (spec * spec)
    rows = s.steps(1500)
    np.testing.assert_array_equal(rows.astype(np.int64), ro.astype(np.int64))
    assert rel(s.X(), so.X()) <= 1e-10
