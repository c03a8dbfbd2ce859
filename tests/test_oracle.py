"""CPU: pin the oracle (oracle/axb_oracle.c) before trusting it.

1. against the committed golden vectors made by the UNMODIFIED reference
   (tests/golden/make_golden.py → oracle/_ref/libaxbref.so);
2. live against oracle/_ref where it is present (this container; GPU boxes that
   received the prebuilt .so);
3. the reference's own known-answer tests (proj/tests/test_solver.cpp).
Bitwise equality is required throughout.
"""
import ctypes as C
import hashlib
import os

import numpy as np
import pytest

import oracle_lib as O

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def gold(name):
    return np.load(os.path.join(GOLD, name))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def c1(orc):
    return O.generate(orc, 7, 500, 100, 80, 400)


# ---------------------------------------------------------------- golden vectors
def test_rng_streams_match_reference(orc):
    g = gold("rng.npz")
    for i, sd in enumerate(g["seeds"]):
        r = O.Rng(); orc.rng_init(C.byref(r), int(sd))
        u = np.array([orc.rng_next_u64(C.byref(r)) for _ in range(256)], dtype=np.uint64)
        np.testing.assert_array_equal(u, g["u64"][i])
        r2 = O.Rng(); orc.rng_init(C.byref(r2), int(sd))
        gs = np.array([orc.rng_gauss(C.byref(r2)) for _ in range(256)])
        np.testing.assert_array_equal(gs, g["gauss"][i])
        for t in range(4):
            sub = O.Rng(); orc.rng_substream(C.byref(r), t, C.byref(sub))
            assert sub.seed == int(g["substream_seeds"][i][t])


def test_generate_config1_matches_reference(c1):
    g = gold("gen_c1.npz")
    A, B, X, Cm = c1
    assert sha(A) == str(g["sha_A"]) and sha(B) == str(g["sha_B"])
    assert sha(X) == str(g["sha_X"]) and sha(Cm) == str(g["sha_C"])


@pytest.mark.parametrize("name,tag,theta", [("grbk", O.GRBK, None), ("mwrbk", O.MWRBK, None)])
def test_config1_full_run_matches_reference(orc, c1, name, tag, theta):
    """Config 1 to ‖X−X*‖/‖X*‖ < 1e-6: iterations, trace rows and X bitwise."""
    g = gold(f"run_c1_{name}.npz")
    A, B, X, Cm = c1
    cfg = O.make_config(method=tag, theta=theta, stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=X,
                        seed=42, record_trace=True, max_iter=40000, refresh_interval=1000)
    s = O.Solver(orc, A, B, Cm, None, cfg)
    rep, rows, _, Xf = s.run(40000)
    assert rep.iterations == int(g["iterations"])
    assert rep.alpha == float(g["alpha"])
    assert rep.final_rrn == float(g["final_rrn"])
    np.testing.assert_array_equal(rows.astype(np.uint16), g["rows"])
    np.testing.assert_array_equal(Xf, g["X"])


@pytest.mark.parametrize("name,tag,theta", [("rgrbk025", O.RGRBK, 0.25), ("rbk", O.RBK, None),
                                            ("bk", O.BK, None)])
def test_config1_prefix_matches_reference(orc, c1, name, tag, theta):
    """First 2500 trace rows of the other methods (run() semantics, refresh every 1000)."""
    g = gold(f"run_c1_{name}.npz")
    A, B, X, Cm = c1
    cfg = O.make_config(method=tag, theta=theta, stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=X,
                        seed=42, record_trace=True, max_iter=2500, refresh_interval=1000)
    s = O.Solver(orc, A, B, Cm, None, cfg)
    rep, rows, _, _ = s.run(2500)
    np.testing.assert_array_equal(rows.astype(np.uint16), g["rows"][:2500])


def test_small_system_kats(orc):
    g = gold("kat_small.npz")
    for k in range(3):
        m, p, q, n, seed = (int(v) for v in g[f"s{k}_shape"])
        A, B, X, Cm = O.generate(orc, seed, m, p, q, n)
        for name, tag, theta in [("bk", O.BK, None), ("grbk", O.GRBK, None),
                                 ("mwrbk", O.MWRBK, None), ("rgrbk08", O.RGRBK, 0.8),
                                 ("rbk", O.RBK, None)]:
            cfg = O.make_config(method=tag, theta=theta, stop_kind=O.RESIDUAL_REL, tol=0.0,
                                seed=77, refresh_interval=0)
            s = O.Solver(orc, A, B, Cm, None, cfg)
            np.testing.assert_array_equal(s.steps(30).astype(np.uint16), g[f"s{k}_{name}_rows"])
            np.testing.assert_array_equal(s.X(), g[f"s{k}_{name}_X"])
            assert s.alpha == float(g[f"s{k}_{name}_alpha"])


# ---------------------------------------------------------------- live reference
ref_only = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


@ref_only
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_live_against_reference(orc, seed):
    r = O.ref()
    rng = np.random.default_rng(seed)
    m, p, q, n = (int(v) for v in rng.integers(3, 40, size=4))
    A, B, X, Cm = O.generate(orc, seed, m, p, q, n)
    X0 = rng.standard_normal((p, q))
    for tag, theta in [(O.BK, None), (O.RBK, None), (O.GRBK, None), (O.RGRBK, 0.3),
                       (O.MWRBK, None)]:
        cfg = O.make_config(method=tag, theta=theta, stop_kind=O.RESIDUAL_REL, tol=0.0,
                            seed=seed, refresh_interval=50)
        so = O.Solver(orc, A, B, Cm, X0, cfg)
        sr = O.Solver(r, A, B, Cm, X0, cfg)
        np.testing.assert_array_equal(so.steps(200, True, 50), sr.steps(200, True, 50))
        np.testing.assert_array_equal(so.X(), sr.X())
        np.testing.assert_array_equal(so.R(), sr.R())
        assert so.residual_fro_sq == sr.residual_fro_sq


@ref_only
def test_error_paths_match_reference(orc):
    r = O.ref()
    Z = np.zeros((2, 2)); I2 = np.eye(2)
    for lib in (orc, r):
        with pytest.raises(O.OracleError) as e:
            O.Solver(lib, Z, I2, Z, None, O.make_config())
        assert e.value.code == 2  # DomainError: A is the zero matrix
        with pytest.raises(O.OracleError) as e:
            O.Solver(lib, I2, I2, Z, None, O.make_config(method=O.RGRBK, theta=1.5))
        assert e.value.code == 3  # ConfigError
        A = np.array([[1.0]]); B = np.array([[10.0]]); Cm = np.array([[10.0]])
        with pytest.raises(O.OracleError) as e:
            O.Solver(lib, A, B, Cm, None, O.make_config(method=O.BK, alpha_rule=O.FIXED,
                                                         alpha_value=0.1))
        assert e.value.code == 3  # fixed alpha outside (0, 2/‖B‖²)
        s = O.Solver(lib, A, B, Cm, None, O.make_config(method=O.BK, alpha_rule=O.PAPER,
                                                         tol=1e-12, max_iter=2000))
        with pytest.raises(O.OracleError) as e:
            s.run()
        assert e.value.code == 4  # DivergenceError (solver.hpp:307)


# ---------------------------------------------------------------- reference KATs
def kat_solver(orc, A, r_sq, seed=0):
    Cm = np.sqrt(np.asarray(r_sq, dtype=np.float64)).reshape(-1, 1)
    return O.Solver(orc, A, np.array([[1.0]]), Cm, None,
                    O.make_config(method=O.GRBK, alpha_rule=O.FIXED, alpha_value=0.5,
                                  stop_kind=O.RESIDUAL_REL, tol=0.0, seed=seed,
                                  refresh_interval=0))


def test_kat_single_entry_step(orc):
    """test_solver.cpp:37-44."""
    s = O.Solver(orc, np.array([[2.0]]), np.array([[1.0]]), np.array([[4.0]]), None,
                 O.make_config(method=O.BK, alpha_rule=O.FIXED, alpha_value=1.0,
                               stop_kind=O.RESIDUAL_REL, tol=0.0, refresh_interval=0))
    s.update_row(0)
    assert s.X()[0, 0] == 2.0 and s.R()[0, 0] == 0.0


def test_kat_thresholds(orc):
    """test_solver.cpp:136-151 (ζ = 0.75, ξ(0.8) = 0.9, θ=½ ≡ GRBK bitwise)."""
    s = kat_solver(orc, np.eye(2), [1.0, 0.0])
    assert s.greedy_threshold(0.5) == pytest.approx(0.75, rel=1e-15)
    assert s.greedy_threshold(0.8) == pytest.approx(0.9, rel=1e-15)
    assert list(s.greedy_index_set(0.5)) == [0]
    t = kat_solver(orc, np.eye(3), [2.0, 2.0, 2.0])
    assert t.max_residual_ratio()[0] == 0  # smallest index on ties (test_solver.cpp:211-218)


def test_kat_greedy_membership_properties(orc):
    """Argmax ∈ set; larger θ never enlarges it (test_solver.cpp:170-209)."""
    for seed in range(10):
        A, B, X, Cm = O.generate(orc, 2000 + seed, 10, 4, 3, 7)
        s = O.Solver(orc, A, B, Cm, None, O.make_config(method=O.GRBK, alpha_rule=O.FIXED,
                                                        alpha_value=0.01, tol=0.0,
                                                        refresh_interval=0))
        am = s.max_residual_ratio()[0]
        sets = [set(s.greedy_index_set(th).tolist()) for th in (0.1, 0.5, 0.9)]
        assert all(am in st for st in sets)
        assert sets[2] <= sets[1] <= sets[0]
