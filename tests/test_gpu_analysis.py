"""GPU parity of the device reference solutions against the oracle.

The device SVD runs the reference's one-sided Jacobi (decomp.hpp:71-109) in
round-robin order, so factors agree with the oracle's cyclic order to rounding,
not bitwise.  Tolerances, stated per check:
  singular values          |Δσ| <= 1e-13·σ_max
  numeric rank, case label  exact
  pseudoinverse            ‖ΔP‖_F <= 1e-11·‖P‖_F
  X* / bk_limit            ‖ΔX‖_F <= 1e-9·(1 + ‖X‖_F)   (the oracle's full-rank
                           cases go through normal equations + LU, the device
                           through the SVD: they agree to ~cond(A)²·ε)
  rrn                      1e-13 relative
Size-independent properties (A·X*·B = C, X* ⟂ null spaces, recovery of the
generating X) cover BASELINE config sizes the oracle cannot finish.
"""
import os

import numpy as np
import pytest

import oracle_lib as O
from configs import config2, config3_rank_deficient

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "analysis.npz")


@pytest.fixture(scope="module")
def P():
    import paper_2408_05444_b200 as P
    assert P.device_available(), "no CUDA device"
    return P


@pytest.fixture(scope="module")
def an():
    return O.Analysis(O.oracle())


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_svd_against_oracle(P, an, gold):
    for name in gold["svd_names"]:
        M = gold[f"svd_{name}_M"]
        f = P.svd(M)
        U, s, V, rank = an.svd(M)
        assert f.numeric_rank == rank, name
        assert np.max(np.abs(f.singular_values - s)) <= 1e-13 * s[0], name
        r = len(s)
        assert np.linalg.norm(f.U.T @ f.U - np.eye(r)) <= 1e-10, name  # test_decomp.cpp:19-22
        assert np.linalg.norm(f.V.T @ f.V - np.eye(r)) <= 1e-10, name
        rec = (f.U * f.singular_values) @ f.V.T
        assert np.linalg.norm(rec - M) <= 1e-10 * max(np.linalg.norm(M), 1.0), name
        # singular vectors of simple, solid σ agree with the oracle up to sign
        for k in range(rank):
            gap = min([abs(s[k] - s[j]) for j in range(r) if j != k] or [1.0])
            if gap > 1e-6 * s[0]:
                sg = np.sign(f.V[:, k] @ V[:, k])
                assert np.linalg.norm(sg * f.V[:, k] - V[:, k]) <= 1e-9, (name, k)
                assert np.linalg.norm(sg * f.U[:, k] - U[:, k]) <= 1e-9, (name, k)


def test_pseudoinverse_against_oracle(P, an, gold):
    for name in gold["svd_names"]:
        M = gold[f"svd_{name}_M"]
        assert rel(P.pseudoinverse(M), gold[f"svd_{name}_pinv"]) <= 1e-11, name
    d = np.array([[2.0, 0.0], [0.0, 0.0]])  # test_decomp.cpp:78-83
    assert np.linalg.norm(P.pseudoinverse(d) - np.array([[0.5, 0], [0, 0]])) <= 1e-12
    assert np.linalg.norm(P.pseudoinverse(np.eye(4)) - np.eye(4)) <= 1e-12
    M = gold["svd_u33x20_M"]
    assert rel(P.pseudoinverse(M, 0.5), an.pseudoinverse(M, 0.5)) <= 1e-11


def test_reference_solution_against_oracle(P, gold):
    for name in gold["names"]:
        A, B, Cm = (gold[f"rs_{name}_{k}"] for k in "ABC")
        tol = float(gold[f"rs_{name}_tol"])
        code = int(gold[f"rs_{name}_code"])
        if code:
            with pytest.raises(P.DomainError, match="system is not consistent"):
                P.reference_solution(A, B, Cm, tol)
            continue
        r = P.reference_solution(A, B, Cm, tol)
        X = gold[f"rs_{name}_X"]
        assert int(r.kind) == int(gold[f"rs_{name}_kind"]), name
        assert np.linalg.norm(r.X_star - X) <= 1e-9 * (1 + np.linalg.norm(X)), name
        assert r.residual_check <= 1e-8 * (1 + np.linalg.norm(Cm)), name
        if f"rs_{name}_bk" in gold:
            bk = P.bk_limit(A, B, Cm, gold[f"rs_{name}_X0"])
            ref = gold[f"rs_{name}_bk"]
            assert np.linalg.norm(bk - ref) <= 1e-9 * (1 + np.linalg.norm(ref)), name


def test_live_random_against_oracle(P, an):
    rng = np.random.default_rng(11)
    for m, p, q, n, deficient in [(30, 12, 10, 25, False), (9, 20, 18, 7, False),
                                  (40, 16, 16, 40, True), (17, 17, 13, 13, False)]:
        A = rng.standard_normal((m, p))
        B = rng.standard_normal((q, n))
        if deficient:
            A[:, -3:] = A[:, :3] @ rng.standard_normal((3, 3))
            B[-2:] = rng.standard_normal((2, 2)) @ B[:2]
        Cm = A @ rng.standard_normal((p, q)) @ B
        X0 = rng.standard_normal((p, q))
        xo, ko, _ = an.reference_solution(A, B, Cm)
        r = P.reference_solution(A, B, Cm)
        assert int(r.kind) == ko
        assert np.linalg.norm(r.X_star - xo) <= 1e-9 * (1 + np.linalg.norm(xo))
        bo = an.bk_limit(A, B, Cm, X0)
        assert np.linalg.norm(P.bk_limit(A, B, Cm, X0) - bo) <= 1e-9 * (1 + np.linalg.norm(bo))
        assert P.rrn(r.X_star, xo) == pytest.approx(an.rrn(r.X_star, xo), rel=1e-13, abs=1e-300)


def test_rank_deficient_completion(P, gold):
    M = gold["svd_dupcols_M"]  # 9×6, rank 3: U's last three columns are completed
    f = P.svd(M)
    assert f.numeric_rank == 3
    assert np.linalg.norm(f.U.T @ f.U - np.eye(6)) <= 1e-10
    assert np.linalg.norm((f.U * f.singular_values) @ f.V.T - M) <= 1e-10 * np.linalg.norm(M)
    U, s, V, rank = O.Analysis(O.oracle()).svd(M)
    # the completed columns are the same projections of e_0, e_1, … (up to rounding)
    assert np.linalg.norm(f.U[:, 3:] - U[:, 3:]) <= 1e-9
    Mt = np.ascontiguousarray(M.T)  # wide: completion lands in V
    g = P.svd(Mt)
    assert np.linalg.norm(g.V.T @ g.V - np.eye(6)) <= 1e-10


def test_errors(P):
    with pytest.raises(P.ShapeError):
        P.svd(np.zeros((0, 3)))
    with pytest.raises(P.DecompositionError, match="Jacobi sweeps exceeded cap"):
        P.svd(np.random.default_rng(0).standard_normal((6, 4)), max_sweeps=1)
    with pytest.raises(P.DomainError, match="zero reference"):
        P.rrn(np.ones((2, 2)), np.zeros((2, 2)))
    assert P.rrn(np.eye(3), np.eye(3)) == 0.0


def test_csr_operands(P, an):
    sp = pytest.importorskip("scipy.sparse")
    rng = np.random.default_rng(5)
    A = sp.random(30, 12, density=0.4, random_state=1, format="csr") + sp.eye(30, 12, format="csr")
    B = sp.random(10, 24, density=0.4, random_state=2, format="csr") + sp.eye(10, 24, format="csr")
    Ad, Bd = A.toarray(), B.toarray()
    Cm = Ad @ rng.standard_normal((12, 10)) @ Bd
    r = P.reference_solution(A.tocsr(), B.tocsr(), Cm)
    xo, ko, _ = an.reference_solution(Ad, Bd, Cm)
    assert int(r.kind) == ko and np.linalg.norm(r.X_star - xo) <= 1e-9 * (1 + np.linalg.norm(xo))


def test_config2_recovers_generator(P):
    """Config 2 (A 2000×500, B 400×2000, σ log-spaced 1..1e-2): unique X* = X."""
    A, B, Xs, Cm = config2(seed=3)
    r = P.reference_solution(A, B, Cm)
    assert r.kind == P.ReferenceCase.UniqueFullRank
    assert np.linalg.norm(r.X_star - Xs) <= 1e-8 * np.linalg.norm(Xs)
    assert r.residual_check <= 1e-8 * (1 + np.linalg.norm(Cm))


def test_config3_analogue_bk_limit(P):
    """The rank-deficient config-3 analogue: bk_limit = A⁺CB⁺ + X0 − A⁺AX0BB⁺ (numpy)."""
    A, B, Cm, X0, target = config3_rank_deficient(seed=4)
    got = P.bk_limit(A, B, Cm, X0)
    assert np.linalg.norm(got - target) <= 1e-8 * np.linalg.norm(target)
    r = P.reference_solution(A, B, Cm)
    assert r.kind == P.ReferenceCase.LeastNormGeneral
    # least norm: X* lies in row(A)ᵀ ⊗ col(B) — invariant under the projector
    Ap, Bp = np.linalg.pinv(A, rcond=1e-10), np.linalg.pinv(B)
    X = r.X_star
    assert np.linalg.norm(Ap @ A @ X @ B @ Bp - X) <= 1e-8 * np.linalg.norm(X)


@pytest.mark.timeout(900)
def test_config3_full_size_recovery(P):
    """BASELINE config 3 sizes (A 8192×2048, B 2048×8192, Gaussian): the device
    X* recovers the generating X (unique solution) — size-independent check."""
    rng = np.random.default_rng(8)
    m, p, q, n = 8192, 2048, 2048, 8192
    A = rng.standard_normal((m, p))
    B = rng.standard_normal((q, n))
    Xs = rng.standard_normal((p, q))
    Cm = (A @ Xs) @ B
    r = P.reference_solution(A, B, Cm)
    sa, sb, ms = P.analysis.last_stats()
    print(f"config3 reference_solution: sweeps {sa}/{sb}, device {ms:.1f} ms")
    assert r.kind == P.ReferenceCase.UniqueFullRank
    assert np.linalg.norm(r.X_star - Xs) <= 1e-8 * np.linalg.norm(Xs)


def test_benchmark_pool_computes_references(P, an):
    """analysis.hpp:261-264: with no X_star the harness solves for it first — on
    the device here; trial iteration counts match the oracle run against the
    oracle's own reference_solution."""
    from paper_2408_05444_b200 import pool

    orc = O.oracle()
    A, B, X, Cm = O.generate(orc, 41, 120, 30, 20, 90)
    probs = [pool.BenchProblem("p0", A, B, Cm, None)]
    methods = [P.Method.rbk(), P.Method.grbk()]
    opt = pool.BenchmarkOptions(trials=2, seed=9, tol=1e-12, jobs=4)
    rows = pool.benchmark(probs, methods, opt)
    xo, _, _ = an.reference_solution(A, B, Cm)
    for r in rows:
        tag = {"rbk": O.RBK, "grbk": O.GRBK}[r.method]
        its = []
        for t in range(2):
            cfg = O.make_config(method=tag, stop_kind=O.SOLUTION_RRN, tol=1e-12, reference=xo,
                                seed=pool.substream_seed(9, t))
            rep, _, _, _ = O.Solver(orc, A, B, Cm, None, cfg).run(0)
            its.append(rep.iterations)
        assert r.failures == 0 and abs(r.it_mean - np.mean(its)) <= 2.0, (r, its)
