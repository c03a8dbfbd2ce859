"""CPU, world_size 2 over gloo: the row-sharded decomposition (one grouped
allgather of the ‖R_l‖² slices and shard records, every rank selecting over the
global rows with the shared draw, owner pack allreduce, column-split y/z,
row-split X: four exchanges per iteration) reproduces the single-process
oracle's rows and iterates.
Runs here without a GPU; the CUDA path of the same schedule is exercised on a
1-rank NCCL communicator by tests/test_gpu_parity.py::test_sharded_mode_one_rank."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle_lib as O

STEPS = 300


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, tag, theta, out_q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import shard_sim

        orc = O.oracle()
        A, B, X, Cm = O.generate(orc, 7, 500, 100, 80, 400)
        cfg = O.make_config(method=tag, theta=theta, stop_kind=O.RESIDUAL_REL, tol=0.0,
                            seed=42, refresh_interval=0)
        so = O.Solver(orc, A, B, Cm, None, cfg)
        alpha = so.alpha
        sh = shard_sim.Shard(A, B, Cm, np.zeros((100, 80)), tag, theta if theta else 0.5, alpha,
                             42, world, rank)
        sh.records()
        rows = [sh.step() for _ in range(STEPS)]
        Xg = sh.gather_X()
        if rank == 0:
            ro = so.steps(STEPS)
            out_q.put((np.array(rows), ro.astype(np.int64), Xg, so.X()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tag,theta", [(O.GRBK, None), (O.MWRBK, None), (O.RBK, None),
                                       (O.BK, None), (O.RGRBK, 0.3)])
def test_two_rank_sharded_schedule_matches_oracle(tag, theta):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tag, theta, q)) for r in range(2)]
    for p in procs:
        p.start()
    rows, ro, Xg, Xo = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mism = np.nonzero(rows != ro)[0]
    assert mism.size == 0, f"first mismatch at step {mism[:5]}"
    assert np.linalg.norm(Xg - Xo) / np.linalg.norm(Xo) <= 1e-10
