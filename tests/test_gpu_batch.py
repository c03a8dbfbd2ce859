"""GPU: many independent solves in one batch (axb_solvers_run / run_many).

Each handle in a batch must end exactly where the oracle's run() ends: same
iteration count (±2, the run-to-tolerance bar of test_gpu_parity.py — the
batched kernel sums ‖R‖² in a different tree order than the cooperative one)
and X within 1e-10 of the oracle's X at that point for deterministic
selections.  Mixed batches cover the paths around the batched kernel: a
graph-path handle (run on its own launches), a max_iter stop, an
already-converged start and a zero residual.
"""
import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu

TAGS = [(O.GRBK, None), (O.MWRBK, None), (O.RGRBK, 0.25), (O.RBK, None), (O.BK, None)]


def method(axb, tag, theta):
    return {O.BK: axb.Method.bk(), O.RBK: axb.Method.rbk(), O.GRBK: axb.Method.grbk(),
            O.RGRBK: axb.Method.rgrbk(theta if theta is not None else 0.5),
            O.MWRBK: axb.Method.mwrbk()}[tag]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def oracle_run(orc, A, B, Cm, X0, tag, theta, seed, Xs, tol, max_iter=200000, refresh=1000):
    cfg = O.make_config(method=tag, theta=theta, stop_kind=O.SOLUTION_RRN, tol=tol, reference=Xs,
                        seed=seed, max_iter=max_iter, refresh_interval=refresh)
    rep, _, _, X = O.Solver(orc, A, B, Cm, X0, cfg).run(0)
    return rep, X


def test_run_many_matches_oracle(axb, orc):
    systems = [O.generate(orc, 60 + k, 120, 30, 20, 90) for k in range(3)]
    handles, expect = [], []
    for k, (A, B, Xs, Cm) in enumerate(systems):
        for tag, theta in TAGS:
            seed = 11 * k + tag
            cfg = axb.SolveConfig(method=method(axb, tag, theta),
                                  stop=axb.StopRule.solution_rrn(1e-12, Xs), seed=seed)
            handles.append(axb.Solver(A, B, Cm, None, cfg))
            expect.append(oracle_run(orc, A, B, Cm, None, tag, theta, seed, Xs, 1e-12))
    reps = axb.run_many(handles)
    for h, rep, (orep, oX), (tag, _) in zip(handles, reps, expect, TAGS * len(systems)):
        assert rep.terminated_by == axb.Terminated.Tolerance
        assert abs(rep.iterations - orep.iterations) <= 2, (tag, rep.iterations, orep.iterations)
        assert rep.final_rrn <= 1e-12
        if rep.iterations == orep.iterations:
            assert rel(rep.X, oX) <= 1e-6  # both at rrn ≤ 1e-12 of the same X*
    # the batch leaves each handle exactly as its own run() would
    for h, rep in zip(handles, reps):
        assert h.iteration() == rep.iterations


def test_run_many_deterministic_sequence_and_x(axb, orc):
    """MWRBK / BK / fixed budget: X after the same iterations within 1e-10."""
    A, B, Xs, Cm = O.generate(orc, 77, 300, 60, 40, 200)
    handles, expect = [], []
    for tag in (O.MWRBK, O.BK, O.GRBK):
        cfg = axb.SolveConfig(method=method(axb, tag, None),
                              stop=axb.StopRule.solution_rrn(0.0, Xs), seed=5, max_iter=3000)
        handles.append(axb.Solver(A, B, Cm, None, cfg))
        expect.append(oracle_run(orc, A, B, Cm, None, tag, None, 5, Xs, 0.0, max_iter=3000))
    for rep, (orep, oX) in zip(axb.run_many(handles), expect):
        assert rep.iterations == orep.iterations == 3000
        assert rep.terminated_by == axb.Terminated.MaxIter
        assert rel(rep.X, oX) <= 1e-10


def test_run_many_mixed_paths(axb, orc, monkeypatch):
    A, B, Xs, Cm = O.generate(orc, 91, 120, 30, 20, 90)
    mk = lambda **kw: axb.SolveConfig(method=axb.Method.grbk(),  # noqa: E731
                                      stop=axb.StopRule.solution_rrn(1e-12, Xs), seed=3, **kw)
    small = axb.Solver(A, B, Cm, None, mk())
    budget = axb.Solver(A, B, Cm, None, mk(max_iter=500))
    done = axb.Solver(A, B, Cm, Xs, mk())  # X0 = X*: converged before the first step
    monkeypatch.setenv("AXB_PERSIST", "0")
    graph = axb.Solver(A, B, Cm, None, mk())  # graph path: runs on its own launches
    monkeypatch.delenv("AXB_PERSIST")
    zero = axb.Solver(A, B, np.zeros_like(Cm), None,
                      axb.SolveConfig(method=axb.Method.mwrbk(), stop=axb.StopRule.residual_rel(0.0),
                                      max_iter=100))
    reps = axb.run_many([small, budget, done, graph, zero])
    orep, _ = oracle_run(orc, A, B, Cm, None, O.GRBK, None, 3, Xs, 1e-12)
    assert abs(reps[0].iterations - orep.iterations) <= 2
    assert abs(reps[3].iterations - orep.iterations) <= 2
    assert reps[1].iterations == 500 and reps[1].terminated_by == axb.Terminated.MaxIter
    assert reps[2].iterations == 0 and reps[2].terminated_by == axb.Terminated.Tolerance
    assert reps[4].iterations == 0  # ‖R‖² = 0 ends the loop (solver.hpp:347)


def test_run_many_rejects_bad_batches(axb, orc):
    A, B, Xs, Cm = O.generate(orc, 5, 60, 20, 10, 40)
    cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(1e-12, Xs))
    h = axb.Solver(A, B, Cm, None, cfg)
    with pytest.raises(axb.ConfigError, match="duplicate"):
        axb.run_many([h, h])
    assert axb.run_many([]) == []


def test_benchmark_pool_batched_equals_threaded(axb, orc):
    from paper_2408_05444_b200 import pool

    probs = []
    for k, seed in enumerate((31, 32)):
        A, B, X, Cm = O.generate(orc, seed, 120, 30, 20, 90)
        probs.append(pool.BenchProblem(f"p{k}", A, B, Cm, X))
    methods = [axb.Method.rbk(), axb.Method.grbk(), axb.Method.mwrbk()]
    rb = pool.benchmark(probs, methods, pool.BenchmarkOptions(trials=4, seed=5, tol=1e-12))
    rt = pool.benchmark(probs, methods,
                        pool.BenchmarkOptions(trials=4, seed=5, tol=1e-12, batched=False, jobs=4))
    for a, b in zip(rb, rt):
        assert (a.problem_id, a.method, a.failures) == (b.problem_id, b.method, b.failures)
        assert abs(a.it_mean - b.it_mean) <= 2.0
