"""GPU: the reference's own solver test cases, run through the C-ABI.

Each test restates one TEST_CASE of proj/tests/test_solver.cpp (cited per test)
on the device path; the reference's random fixtures (testsup::random_gaussian,
mt19937) are replaced by seeded numpy Gaussians of the same shapes — the cases
are properties, not golden values.  The tiny systems run on the persistent
latency body by default; the property cases that iterate also run on the
general persistent body and on the graph path (`path` fixture).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def gauss(rows, cols, seed):
    return np.random.default_rng(seed).standard_normal((rows, cols))


def fixed(axb, method, alpha, max_iter=1000, **kw):
    """fixed_alpha_config (test_solver.cpp:13-22)."""
    return axb.SolveConfig(method=method, alpha_rule=axb.AlphaRule.Fixed, alpha_value=alpha,
                           stop=axb.StopRule.residual_rel(0.0), max_iter=max_iter,
                           refresh_interval=0, **kw)


@pytest.fixture(params=["persistent", "general", "graph"])
def path(request, monkeypatch):
    if request.param == "graph":
        monkeypatch.setenv("AXB_PERSIST", "0")
    if request.param == "general":
        monkeypatch.setenv("AXB_PERSIST_LAT", "0")
    return request.param


def test_zero_residual_row_is_fixed_point(axb):
    """test_solver.cpp:46-57."""
    A = np.eye(2)
    B = np.array([[1.0]])
    C = A @ np.array([[1.0], [4.0]]) @ B
    s = axb.Solver(A, B, C, np.array([[1.0], [0.0]]), fixed(axb, axb.Method.bk(), 1.0))
    x0, r0 = s.X(), s.R()
    s.update_row(0)
    assert np.array_equal(s.X(), x0)
    assert np.array_equal(s.R(), r0)


def test_incremental_residual_tracks_recomputation(axb, path):
    """test_solver.cpp:59-69: 50 RBK steps, ‖R_inc − (C − AXB)‖_F ≤ 1e-10."""
    A, B, X = gauss(6, 4, 301), gauss(4, 5, 302), gauss(4, 4, 303)
    s = axb.Solver(A, B, A @ X @ B, np.zeros((4, 4)),
                   fixed(axb, axb.Method.rbk(), 0.02, 50, seed=5))
    for _ in range(50):
        s.step()
    assert s.residual_drift() <= 1e-10


def test_cyclic_selection_sweeps_rows_in_order(axb):
    """test_solver.cpp:71-86."""
    B = gauss(2, 2, 312)
    A = gauss(3, 2, 311)
    s = axb.Solver(A, B, A @ gauss(2, 2, 313) @ B, np.zeros((2, 2)),
                   fixed(axb, axb.Method.bk(), 0.05))
    assert [s.select_cyclic() for _ in range(4)] == [0, 1, 2, 0]
    A1 = gauss(1, 2, 314)
    s1 = axb.Solver(A1, B, A1 @ gauss(2, 2, 315) @ B, np.zeros((2, 2)),
                    fixed(axb, axb.Method.bk(), 0.05))
    assert [s1.select_cyclic() for _ in range(2)] == [0, 0]


def test_rbk_selection_follows_row_norm_distribution(axb):
    """test_solver.cpp:88-117 (frequencies over 10⁴ draws of the device stream)."""
    B = np.eye(2)
    A0 = np.array([[0.0, 0.0], [2.0, 1.0], [0.0, 0.0]])
    s0 = axb.Solver(A0, B, A0 @ gauss(2, 2, 321) @ B, np.zeros((2, 2)),
                    fixed(axb, axb.Method.rbk(), 0.5))
    assert all(s0.select_rbk() == 1 for _ in range(50))
    A1 = np.eye(2)
    s1 = axb.Solver(A1, B, A1 @ gauss(2, 2, 322) @ B, np.zeros((2, 2)),
                    fixed(axb, axb.Method.rbk(), 0.5, seed=17))
    hits = sum(s1.select_rbk() == 0 for _ in range(10000)) / 10000.0
    assert 0.46 <= hits <= 0.54
    A2 = np.array([[np.sqrt(3.0), 0.0], [1.0, 0.0]])
    s2 = axb.Solver(A2, B, A2 @ gauss(2, 2, 323) @ B, np.zeros((2, 2)),
                    fixed(axb, axb.Method.rbk(), 0.5, seed=29))
    hits = sum(s2.select_rbk() == 0 for _ in range(10000)) / 10000.0
    assert 0.71 <= hits <= 0.79


def test_threshold_collapses_when_all_ratios_equal(axb):
    """test_solver.cpp:146-150: R = A (B = I, X0 = 0) ⇒ ζ·‖A‖²_F = 1."""
    As = gauss(3, 3, 332)
    s = axb.Solver(As, np.eye(3), As, np.zeros((3, 3)), fixed(axb, axb.Method.grbk(), 0.5))
    a_fro = float(np.sum(As * As))
    assert s.grbk_threshold() * a_fro == pytest.approx(1.0, rel=1e-12)
    assert s.grbk_threshold() >= 1.0 / a_fro - 1e-18


def test_threshold_times_frobenius_mass_at_least_one(axb):
    """test_solver.cpp:154-162."""
    for seed in range(10):
        A, B = gauss(8, 5, 1000 + seed), gauss(5, 6, 1100 + seed)
        s = axb.Solver(A, B, A @ gauss(5, 5, 1200 + seed) @ B, np.zeros((5, 5)),
                       fixed(axb, axb.Method.grbk(), 0.01))
        assert s.grbk_threshold() * s.a_fro_sq() >= 1.0 - 1e-12


def test_argmax_row_belongs_to_greedy_set(axb):
    """test_solver.cpp:170-190: argmax ∈ 𝒥_k(θ) and every member meets the inequality."""
    for seed in range(20):
        A, B = gauss(10, 4, 2000 + seed), gauss(3, 7, 2100 + seed)
        s = axb.Solver(A, B, A @ gauss(4, 3, 2200 + seed) @ B, np.zeros((4, 3)),
                       fixed(axb, axb.Method.grbk(), 0.01))
        r_sq, a_sq, r_fro = s.residual_row_sq(), s.a_row_sq(), s.residual_fro_sq()
        for theta in (0.1, 0.5, 0.9):
            members = s.greedy_index_set(theta)
            argmax = s.max_residual_ratio()[0]
            assert argmax in members
            zeta = s.greedy_threshold(theta)
            for i in members:
                assert i == argmax or r_sq[i] >= zeta * a_sq[i] * r_fro


def test_larger_theta_never_enlarges_the_set(axb):
    """test_solver.cpp:192-209."""
    for seed in range(10):
        A, B = gauss(12, 5, 3000 + seed), gauss(4, 6, 3100 + seed)
        s = axb.Solver(A, B, A @ gauss(5, 4, 3200 + seed) @ B, np.zeros((5, 4)),
                       fixed(axb, axb.Method.grbk(), 0.01))
        low, mid, high = (set(s.greedy_index_set(t)) for t in (0.1, 0.5, 0.9))
        assert high <= mid <= low


def test_mwrbk_selected_ratio_is_the_exact_maximum(axb):
    """test_solver.cpp:220-232."""
    for seed in range(10):
        A, B = gauss(9, 4, 4000 + seed), gauss(4, 5, 4100 + seed)
        s = axb.Solver(A, B, A @ gauss(4, 4, 4200 + seed) @ B, np.zeros((4, 4)),
                       fixed(axb, axb.Method.mwrbk(), 0.01))
        pick = s.select_mwrbk()
        r_sq, a_sq = s.residual_row_sq(), s.a_row_sq()
        ratio = r_sq[pick] / a_sq[pick]
        assert np.all(ratio >= r_sq / a_sq)
        assert ratio == s.max_residual_ratio()[1]


def test_selection_invariant_under_residual_scaling(axb):
    """test_solver.cpp:234-247: C ↦ 4C (exact) leaves every selection set unchanged."""
    A, B = gauss(8, 4, 5001), gauss(3, 5, 5002)
    C = A @ gauss(4, 3, 5003) @ B
    s = axb.Solver(A, B, C, np.zeros((4, 3)), fixed(axb, axb.Method.grbk(), 0.01, seed=8))
    s4 = axb.Solver(A, B, 4.0 * C, np.zeros((4, 3)), fixed(axb, axb.Method.grbk(), 0.01, seed=8))
    for theta in (0.1, 0.5, 0.9):
        assert s.greedy_index_set(theta) == s4.greedy_index_set(theta)
    assert s.select_mwrbk() == s4.select_mwrbk()
    assert s.grbk_threshold() * 16.0 == pytest.approx(s4.grbk_threshold() * 16.0)


def test_solve_trivial_system_and_solved_start(axb, path):
    """test_solver.cpp:249-265."""
    A, B, C = np.array([[2.0]]), np.array([[1.0]]), np.array([[4.0]])
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Fixed, alpha_value=1.0,
                          stop=axb.StopRule.residual_rel(1e-12))
    rep = axb.solve(A, B, C, np.zeros((1, 1)), cfg)
    assert rep.iterations == 1
    assert rep.terminated_by == axb.Terminated.Tolerance
    assert rep.X[0, 0] == pytest.approx(2.0)
    rep0 = axb.solve(A, B, C, np.array([[2.0]]), cfg)
    assert rep0.iterations == 0
    assert rep0.terminated_by == axb.Terminated.Tolerance


def test_grbk_and_rgrbk_half_share_the_trajectory(axb, path):
    """test_solver.cpp:267-286 (acceptance C3): identical traces and X."""
    A, B = gauss(12, 5, 6001), gauss(4, 9, 6002)
    C = A @ gauss(5, 4, 6003) @ B
    mk = lambda m: axb.SolveConfig(method=m, stop=axb.StopRule.residual_rel(1e-10),  # noqa: E731
                                   max_iter=400, seed=77, record_trace=True)
    g = axb.solve(A, B, C, np.zeros((5, 4)), mk(axb.Method.grbk()))
    r = axb.solve(A, B, C, np.zeros((5, 4)), mk(axb.Method.rgrbk(0.5)))
    assert len(g.trace) == len(r.trace) > 0
    assert [t.selected_row for t in g.trace] == [t.selected_row for t in r.trace]
    assert np.max(np.abs(g.X - r.X)) <= 1e-15


def test_bk_keeps_the_projection_residue_constant(axb, path):
    """test_solver.cpp:288-316: rank-deficient A and B, X − A⁺(AXB)B⁺ is invariant."""
    g = gauss(3, 6, 6101)
    A = np.vstack([g, g])
    B = gauss(4, 5, 6102)
    C = A @ gauss(6, 4, 6103) @ B
    X0 = 1e-5 * np.eye(6, 4)
    Ap, Bp = np.linalg.pinv(A), np.linalg.pinv(B)
    residue = lambda x: x - Ap @ (A @ x @ B) @ Bp  # noqa: E731
    expected = residue(X0)
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Safe,
                          stop=axb.StopRule.residual_rel(0.0), max_iter=0, refresh_interval=0)
    s = axb.Solver(A, B, C, X0, cfg)
    assert np.linalg.norm(residue(s.X()) - expected) <= 1e-8
    for k in range(100):
        s.step()
        if k in (9, 99):
            assert np.linalg.norm(residue(s.X()) - expected) <= 1e-8


def test_bk_error_never_increases(axb, path):
    """test_solver.cpp:318-343: ‖X_k − X*‖ and ‖X_k − X_lim‖ are non-increasing."""
    A, B = gauss(7, 4, 6201), gauss(3, 6, 6202)
    C = A @ gauss(4, 3, 6203) @ B
    X0 = 0.3 * np.eye(4, 3)
    Ap, Bp = np.linalg.pinv(A), np.linalg.pinv(B)
    x_star = Ap @ C @ Bp
    limit = x_star + X0 - Ap @ A @ X0 @ B @ Bp  # bk_limit (analysis.hpp:95-104)
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Safe,
                          stop=axb.StopRule.residual_rel(0.0), max_iter=0, refresh_interval=0)
    s = axb.Solver(A, B, C, X0, cfg)
    prev_s = np.sum((s.X() - x_star) ** 2)
    prev_l = np.sum((s.X() - limit) ** 2)
    for _ in range(300):
        s.step()
        cur_s, cur_l = np.sum((s.X() - x_star) ** 2), np.sum((s.X() - limit) ** 2)
        assert cur_s <= prev_s + 1e-12
        assert cur_l <= prev_l + 1e-12
        prev_s, prev_l = cur_s, cur_l


def test_zero_rows_are_skipped_by_every_rule(axb, path):
    """test_solver.cpp:345-366."""
    A = np.array([[1.0, 2.0], [0.0, 0.0], [2.0, 1.0]])
    B = gauss(2, 3, 6301)
    C = A @ gauss(2, 2, 6302) @ B
    cfg = lambda m: axb.SolveConfig(method=m, alpha_rule=axb.AlphaRule.Safe,  # noqa: E731
                                    stop=axb.StopRule.residual_rel(1e-10), max_iter=5000)
    rep = axb.solve(A, B, C, np.zeros((2, 2)), cfg(axb.Method.bk()))
    assert rep.terminated_by == axb.Terminated.Tolerance
    assert rep.skipped_zero_rows > 0
    greedy = axb.Solver(A, B, C, np.zeros((2, 2)), cfg(axb.Method.grbk()))
    for _ in range(50):
        if not greedy.residual_fro_sq() > 1e-20:
            break
        assert greedy.step() != 1
    rand = axb.Solver(A, B, C, np.zeros((2, 2)), cfg(axb.Method.rbk()))
    assert all(rand.select_rbk() != 1 for _ in range(50))


def test_all_zero_matrix_is_rejected(axb):
    """test_solver.cpp:368-374."""
    with pytest.raises(axb.DomainError):
        axb.solve(np.zeros((2, 2)), np.eye(2), np.zeros((2, 2)), np.zeros((2, 2)),
                  axb.SolveConfig())


def test_alpha_rules(axb, path):
    """test_solver.cpp:376-395: Fixed outside (0, 2/‖B‖²) → ConfigError; inside
    converges; the Paper rule 1/‖B‖ overshoots here and the guard raises."""
    A, B, C = np.array([[1.0]]), np.array([[10.0]]), np.array([[10.0]])
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Fixed, alpha_value=0.1)
    with pytest.raises(axb.ConfigError):
        axb.solve(A, B, C, np.zeros((1, 1)), cfg)
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Fixed, alpha_value=0.01)
    assert axb.solve(A, B, C, np.zeros((1, 1)), cfg).terminated_by == axb.Terminated.Tolerance
    cfg = axb.SolveConfig(method=axb.Method.bk(), alpha_rule=axb.AlphaRule.Paper,
                          stop=axb.StopRule.residual_rel(1e-12), max_iter=2000)
    with pytest.raises(axb.DivergenceError):
        axb.solve(A, B, C, np.zeros((1, 1)), cfg)


def test_drift_checkpoints_hold_over_long_run(axb, path):
    """test_solver.cpp:405-419: 5000 GRBK steps with a refresh every 1000, no
    InvariantError, residual reduced."""
    A, B = gauss(20, 8, 6401), gauss(6, 15, 6402)
    C = A @ gauss(8, 6, 6403) @ B
    cfg = axb.SolveConfig(method=axb.Method.grbk(), alpha_rule=axb.AlphaRule.Safe,
                          stop=axb.StopRule.residual_rel(0.0), max_iter=5000,
                          refresh_interval=1000, seed=3)
    rep = axb.solve(A, B, C, np.zeros((8, 6)), cfg)
    assert rep.iterations == 5000
    assert rep.final_residual_rel < 1.0
