"""GPU: the row-sharded path with world = 2, 4, 8 on ONE device.

Each rank is a host thread with its own solver handle and stream on cuda:0; the
collectives run through the library's in-process emulation
(axb_nccl_emulated_group: stream sync, host barrier, rank 0 combines, barrier),
so no rank's kernel ever waits on another's (the profiling recipe's rule for
fewer GPUs than ranks).  Everything else is the production sharded path:
column-split y/z, row-split X, the grouped allgather of the ‖R_l‖² slices and
shard records, the selection over the global rows that every rank runs with the
shared xoshiro draw (tie guard included), the owner's row pack, the sharded init
(a_sq, G columns, ‖B‖₂, R0) and checkpoints.  Bar: the oracle's rows and X within
1e-10, as for one GPU.
"""
import threading

import numpy as np
import pytest

import oracle_lib as O

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def method(axb, tag, theta):
    return {O.BK: axb.Method.bk(), O.RBK: axb.Method.rbk(), O.GRBK: axb.Method.grbk(),
            O.RGRBK: axb.Method.rgrbk(theta if theta is not None else 0.5),
            O.MWRBK: axb.Method.mwrbk()}[tag]


def run_ranks(world, fn):
    """fn(rank) on `world` threads; first exception re-raised."""
    out, errs = [None] * world, []

    def body(r):
        try:
            out[r] = fn(r)
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("tag,theta", [(O.GRBK, None), (O.MWRBK, None), (O.RGRBK, 0.3),
                                       (O.RBK, None), (O.BK, None)])
def test_sharded_world_matches_oracle(axb, orc, world, tag, theta):
    from paper_2408_05444_b200 import shard

    m, p, q, n = 512, 96, 40, 200
    A, B, X, Cm = O.generate(orc, 7, m, p, q, n)
    cfg_o = O.make_config(method=tag, theta=theta, seed=42, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=X, refresh_interval=0)
    so = O.Solver(orc, A, B, Cm, None, cfg_o)
    ro = so.steps(600)
    Xo = so.X()
    comms = shard.emulated_comms(world)
    ml = m // world
    try:
        def rank(r):
            cfg = axb.SolveConfig(method=method(axb, tag, theta),
                                  stop=axb.StopRule.solution_rrn(0.0, X), seed=42,
                                  refresh_interval=0)
            s = shard.sharded_solver(np.ascontiguousarray(A[r * ml:(r + 1) * ml]), B,
                                     np.ascontiguousarray(Cm[r * ml:(r + 1) * ml]), None, cfg,
                                     comms[r], world, r)
            rows = s.steps(600)
            Xr = s.X()
            em = s.exact_metric()
            s.checkpoint()
            more = s.steps(100)
            del s
            return rows, Xr, em, more

        res = run_ranks(world, rank)
    finally:
        for c in comms:
            shard.nccl_comm_destroy(c)
    em_o = so.exact_metric()
    so.checkpoint()
    more_o = so.steps(100)
    for rows, Xr, em, more in res:  # every rank reports the global sequence and X
        mism = np.nonzero(rows != ro)[0]
        assert mism.size == 0, f"world {world}: first row mismatch at step {mism[:5]}"
        assert rel(Xr, Xo) <= 1e-10
        np.testing.assert_array_equal(more, more_o)
        assert em == pytest.approx(em_o, rel=1e-8)
    X0r = res[0][1]
    for _, Xr, _, _ in res[1:]:
        np.testing.assert_array_equal(Xr, X0r)


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_world_x_and_run_to_tolerance(axb, orc, world):
    """X after a fixed budget within 1e-10 of the oracle, and run() to
    ‖X−X*‖/‖X*‖ < 1e-6 in the oracle's iteration count ±2 (refresh every 1000)."""
    from paper_2408_05444_b200 import shard

    A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)
    cfg_o = O.make_config(method=O.GRBK, seed=42, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=X, refresh_interval=0)
    so = O.Solver(orc, A, B, Cm, None, cfg_o)
    so.steps(1000)
    comms = shard.emulated_comms(world)
    ml = 500 // world
    try:
        def rank(r):
            sl = slice(r * ml, (r + 1) * ml)
            a, c = np.ascontiguousarray(A[sl]), np.ascontiguousarray(Cm[sl])
            cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X),
                                  seed=42, refresh_interval=0)
            s = shard.sharded_solver(a, B, c, None, cfg, comms[r], world, r)
            s.steps(1000)
            Xr = s.X()
            del s
            cfg = axb.SolveConfig(method=axb.Method.grbk(),
                                  stop=axb.StopRule.solution_rrn(1e-12, X), seed=42,
                                  refresh_interval=1000)
            rep = shard.sharded_solver(a, B, c, None, cfg, comms[r], world, r).run()
            return Xr, rep

        res = run_ranks(world, rank)
    finally:
        for c in comms:
            shard.nccl_comm_destroy(c)
    for Xr, rep in res:
        assert rel(Xr, so.X()) <= 1e-10
        assert rep.terminated_by == axb.Terminated.Tolerance
        assert abs(rep.iterations - 13483) <= 2


def test_sharded_config5_shape_world8(axb, orc):
    """Config 5's aspect ratio at 1/16 scale (A 4096×512, B 512×2048, Gaussian
    scaled as config 5) over 8 emulated ranks: 512 rows per rank, 256-column
    slices of B, 64-row slices of X; 300 GRBK steps match the oracle."""
    from paper_2408_05444_b200 import shard

    m, p, q, n, world = 4096, 512, 512, 2048, 8
    rng = np.random.default_rng(5)
    A = rng.standard_normal((m, p)) / np.sqrt(p)
    B = rng.standard_normal((q, n)) / np.sqrt(n)
    X = rng.standard_normal((p, q))
    Cm = (A @ X) @ B
    cfg_o = O.make_config(method=O.GRBK, seed=42, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=X, refresh_interval=0)
    so = O.Solver(orc, A, B, Cm, None, cfg_o)
    ro = so.steps(300)
    comms = shard.emulated_comms(world)
    ml = m // world
    try:
        def rank(r):
            sl = slice(r * ml, (r + 1) * ml)
            cfg = axb.SolveConfig(method=axb.Method.grbk(), stop=axb.StopRule.solution_rrn(0.0, X),
                                  seed=42, refresh_interval=0)
            s = shard.sharded_solver(np.ascontiguousarray(A[sl]), B, np.ascontiguousarray(Cm[sl]),
                                     None, cfg, comms[r], world, r)
            return s.steps(300), s.X()

        res = run_ranks(world, rank)
    finally:
        for c in comms:
            shard.nccl_comm_destroy(c)
    for rows, Xr in res:
        mism = np.nonzero(rows != ro)[0]
        assert mism.size == 0, f"first row mismatch at step {mism[:5]}"
        assert rel(Xr, so.X()) <= 1e-10


@pytest.mark.parametrize("world", [1, 8])
@pytest.mark.parametrize("tag,theta", [(O.GRBK, None), (O.RGRBK, 0.3)])
def test_sharded_forced_near_tie_walk(axb, orc, world, tag, theta):
    """The near-tie path of the sharded selection.  tie_guard = 2 makes EVERY
    greedy draw take the exact fallback — the reference's sequential member-mass
    walk with upper_bound and the zero-weight walk-back (solver.hpp:243-253,
    rng.hpp:84-99) over the global rows — which a real near-tie takes only when
    the draw lands within 8·m·ε·total of a boundary.  Every rank must still pick
    the oracle's row on every step, and count one walk per draw."""
    from paper_2408_05444_b200 import shard

    m, p, q, n = 1024, 64, 32, 160
    A, B, X, Cm = O.generate(orc, 13, m, p, q, n)
    A[5] = 0.0  # a zero row of A (and of C): never a member
    Cm[5] = 0.0
    k = 300
    cfg_o = O.make_config(method=tag, theta=theta, seed=9, stop_kind=O.SOLUTION_RRN, tol=0.0,
                          reference=X, refresh_interval=0)
    so = O.Solver(orc, A, B, Cm, None, cfg_o)
    ro = so.steps(k)
    comms = shard.emulated_comms(world)
    ml = m // world
    try:
        def rank(r):
            sl = slice(r * ml, (r + 1) * ml)
            cfg = axb.SolveConfig(method=method(axb, tag, theta),
                                  stop=axb.StopRule.solution_rrn(0.0, X), seed=9,
                                  refresh_interval=0)
            s = shard.sharded_solver(np.ascontiguousarray(A[sl]), B, np.ascontiguousarray(Cm[sl]),
                                     None, cfg, comms[r], world, r, tie_guard=2)
            rows = s.steps(k)
            return rows, s.X(), s.selection_stats()

        res = run_ranks(world, rank)
    finally:
        for c in comms:
            shard.nccl_comm_destroy(c)
    for rows, Xr, stats in res:
        mism = np.nonzero(rows != ro)[0]
        assert mism.size == 0, f"first row mismatch at step {mism[:5]}"
        assert rel(Xr, so.X()) <= 1e-10
        assert stats["sequential_walks"] == stats["greedy_selections"] >= k
