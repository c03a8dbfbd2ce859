"""Row-sharded single system over NCCL, host-side plumbing.

One process per GPU.  torch.distributed (any backend; gloo is enough) carries
only the NCCL unique id at start-up; every data-path exchange of the iteration
is an NCCL call the C-ABI library enqueues itself (inside its CUDA graphs):

    y partial  → allreduce (q doubles)      z slice   → allgather (n doubles)
    ‖R_l‖² slice + record → one grouped allgather (m_local + 4 doubles per rank)
    owner row  → allreduce (n + p + 2; only the owner contributes non-zeros)

After the grouped allgather every rank holds the global ‖R_l‖², so every rank
runs the single-GPU selection over the global rows (tie guard and the
reference's sequential walk included) and all ranks agree on the row.

Rows are split into equal contiguous shards (m_global = world·m_local).
"""
from __future__ import annotations

import ctypes as C

from . import _lib
from .errors import CudaError
from .solver import Options, Solver


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    if _lib.load().axb_nccl_unique_id(buf):
        raise CudaError(f"ncclGetUniqueId failed: {_lib.load().axb_last_create_error().decode()}")
    return buf.raw


def nccl_comm_create(nranks: int, uid: bytes, rank: int, device: int) -> int:
    comm = C.c_void_p()
    st = _lib.load().axb_nccl_comm_create(nranks, uid, rank, device, C.byref(comm))
    if st:
        raise CudaError(f"ncclCommInitRank failed: {_lib.load().axb_last_create_error().decode()}")
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    if comm:
        _lib.load().axb_nccl_comm_destroy(C.c_void_p(comm))


def emulated_comms(world: int) -> list:
    """`world` communicators of the in-process collective emulation (test
    infrastructure): one per rank, the ranks being host threads of this process
    on one GPU (axb_nccl_emulated_group)."""
    arr = (C.c_void_p * world)()
    st = _lib.load().axb_nccl_emulated_group(world, arr)
    if st:
        raise CudaError("axb_nccl_emulated_group failed")
    return [arr[i] for i in range(world)]


def init_comm(device: int):
    """Collective over torch.distributed: rank 0 makes the id, all ranks join."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(), dist.get_rank()
    box = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return nccl_comm_create(world, box[0], rank, device), world, rank


def shard_rows(m_global: int, world: int, rank: int):
    if m_global % world:
        raise ValueError("row sharding needs m_global divisible by the world size")
    m = m_global // world
    return rank * m, m


def sharded_solver(A_local, B, C_local, X0, cfg, comm: int, world: int, rank: int,
                   device: int = 0, **opts) -> Solver:
    """Solver over this rank's rows of A and C (B, X0 and cfg.stop.reference full)."""
    m_local = (A_local.__cuda_array_interface__["shape"][0]
               if hasattr(A_local, "__cuda_array_interface__") else len(A_local))
    o = Options(device=device, nccl_comm=comm, world_size=world, rank=rank,
                m_global=m_local * world, row_offset=m_local * rank, **opts)
    return Solver(A_local, B, C_local, X0, cfg, o)
