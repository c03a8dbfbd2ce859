"""Pins the oracle's reference-solution restatement — CPU only.

oracle/axb_oracle.c restates decomp.hpp svd (:113-157, one-sided cyclic Jacobi
:71-109, basis completion :39-65), pseudoinverse (:161-177), lu_solve (:249-279)
and analysis.hpp reference_solution (:48-91), bk_limit (:95-104), rrn (:107-111).
It must be BITWISE equal to the reference on the committed fixtures
(tests/golden/analysis.npz, made by oracle/_ref from the reference headers) and,
where oracle/_ref is built, on fresh random inputs.
"""
import os

import numpy as np
import pytest

import oracle_lib as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "analysis.npz")


@pytest.fixture(scope="module")
def an():
    return O.Analysis(O.oracle())


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def test_svd_matches_golden(an, gold):
    for name in gold["svd_names"]:
        U, s, V, rank = an.svd(gold[f"svd_{name}_M"])
        assert rank == int(gold[f"svd_{name}_rank"]), name
        assert np.array_equal(s, gold[f"svd_{name}_s"]), name
        assert np.array_equal(U, gold[f"svd_{name}_U"]), name
        assert np.array_equal(V, gold[f"svd_{name}_V"]), name
        assert np.array_equal(an.pseudoinverse(gold[f"svd_{name}_M"]), gold[f"svd_{name}_pinv"])


def test_reference_solution_matches_golden(an, gold):
    for name in gold["names"]:
        args = [gold[f"rs_{name}_{k}"] for k in ("A", "B", "C")]
        tol = float(gold[f"rs_{name}_tol"])
        code = int(gold[f"rs_{name}_code"])
        if code:
            with pytest.raises(O.OracleError) as ei:
                an.reference_solution(*args, tol)
            assert ei.value.code == code
            assert str(ei.value) == str(gold[f"rs_{name}_msg"])
            continue
        X, kind, res = an.reference_solution(*args, tol)
        assert kind == int(gold[f"rs_{name}_kind"]), name
        assert np.array_equal(X, gold[f"rs_{name}_X"]), name
        assert res == float(gold[f"rs_{name}_res"]), name
        if f"rs_{name}_bk" in gold:
            bk = an.bk_limit(*args, gold[f"rs_{name}_X0"])
            assert np.array_equal(bk, gold[f"rs_{name}_bk"]), name


def test_reference_solution_properties(an, gold):
    """test_analysis.cpp:24-104 identities, on the restatement."""
    C4 = gold["rs_identity_C"]
    X, kind, _ = an.reference_solution(np.eye(4), np.eye(4), C4)
    assert kind == O.UNIQUE_FULL_RANK and np.linalg.norm(X - C4) <= 1e-10
    A, B, Cm = (gold[f"rs_general_{k}"] for k in "ABC")
    X, kind, _ = an.reference_solution(A, B, Cm)
    assert kind == O.LEAST_NORM_GENERAL
    Ap, Bp = an.pseudoinverse(A), an.pseudoinverse(B)
    rng = np.random.default_rng(3)
    for _ in range(5):  # X* + (Y − A⁺AYBB⁺) solves the system and is never shorter
        Y = rng.standard_normal(X.shape)
        null = Y - Ap @ (A @ Y @ B) @ Bp
        other = X + null
        assert np.linalg.norm(A @ other @ B - Cm) <= 1e-8 * (1 + np.linalg.norm(Cm))
        assert np.sum(other ** 2) == pytest.approx(np.sum(X ** 2) + np.sum(null ** 2), rel=1e-9)
    # zero start → least-norm solution; an exact solution is its own limit
    assert np.linalg.norm(an.bk_limit(A, B, Cm, np.zeros_like(X)) - X) <= 1e-10 * (1 + np.linalg.norm(X))
    assert np.linalg.norm(an.bk_limit(A, B, Cm, X) - X) <= 1e-8 * (1 + np.linalg.norm(X))
    # rrn closed forms (test_analysis.cpp:107-113)
    assert an.rrn(X, X) == 0.0
    assert an.rrn(2 * X, X) == pytest.approx(1.0, rel=1e-12)
    with pytest.raises(O.OracleError) as ei:
        an.rrn(X, np.zeros_like(X))
    assert ei.value.code == O.DOMAIN_ERROR


def test_error_paths(an):
    with pytest.raises(O.OracleError) as ei:
        an.svd(np.zeros((0, 3)))
    assert ei.value.code == O.SHAPE_ERROR
    with pytest.raises(O.OracleError) as ei:  # one sweep cannot diagonalise a 6×4 Gaussian
        an.svd(np.random.default_rng(0).standard_normal((6, 4)), max_sweeps=1)
    assert ei.value.code == O.DECOMPOSITION_ERROR


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_live_against_reference(an, seed):
    ref = O.Analysis(O.ref())
    rng = np.random.default_rng(100 + seed)
    for shape in [(9, 6), (6, 9), (16, 16), (25, 7)]:
        M = rng.standard_normal(shape)
        for a, b in zip(an.svd(M), ref.svd(M)):
            assert np.array_equal(a, b)
    m, p, q, n = [(10, 6, 5, 12), (5, 9, 11, 6), (12, 8, 8, 12)][seed]
    A = rng.standard_normal((m, p))
    if seed == 2:  # rank-deficient A and B
        A[:, -2:] = A[:, :2]
    B = rng.standard_normal((q, n))
    if seed == 2:
        B[-1] = B[0]
    Cm = A @ rng.standard_normal((p, q)) @ B
    X0 = rng.standard_normal((p, q))
    xa, ka, ra = an.reference_solution(A, B, Cm)
    xb, kb, rb = ref.reference_solution(A, B, Cm)
    assert ka == kb and ra == rb and np.array_equal(xa, xb)
    assert np.array_equal(an.bk_limit(A, B, Cm, X0), ref.bk_limit(A, B, Cm, X0))
    with pytest.raises(O.OracleError) as e1:
        an.svd(rng.standard_normal((6, 4)), max_sweeps=1)
    with pytest.raises(O.OracleError) as e2:
        ref.svd(rng.standard_normal((6, 4)), max_sweeps=1)
    assert e1.value.code == e2.value.code == O.DECOMPOSITION_ERROR
    assert str(e1.value) == str(e2.value)
