"""CPU simulation of the row-sharded iteration (test infrastructure).

Mirrors, step for step, what csrc/axb_iter.cu (k_yg_tma/k_zx/k_r_tma in sharded
mode, k_sel1, k_pack) and csrc/axb_solver.cu (enqueue_iteration) do across
ranks, with torch.distributed (gloo) standing in for NCCL — four exchanges per
iteration:

  pack (owner's R_i | A_i | i | coef) → allreduce      y partial (column slice) → allreduce
  z slice → allgather
  local R update → ONE grouped allgather: every shard's ‖R_l‖² slice and record
  then EVERY rank: global ‖R‖², max/argmax in rank order, and the single-GPU
  selection over the global rows (membership, ordered member-mass prefix, one draw
  from the identical xoshiro state, upper_bound and the walk back over zero
  weights, solver.hpp:241-254, rng.hpp:84-99) — all ranks agree with no further
  exchange; the owner fills the pack.

Used by tests/test_shard_gloo.py (world_size 2) against the oracle.
"""
import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

import oracle_lib as O


class Shard:
    def __init__(self, A, B, Cm, X0, method, theta, alpha, seed, world, rank):
        self.world, self.rank = world, rank
        m_g, self.p = A.shape
        self.q, self.n = B.shape
        self.ml = m_g // world
        self.row0 = rank * self.ml
        self.A_g = A  # a_sq of all rows and the owner's A_i (each rank holds its rows)
        self.A = A[self.row0:self.row0 + self.ml].copy()
        self.B = B
        self.C = Cm[self.row0:self.row0 + self.ml].copy()
        self.X = X0.copy()
        nl = -(-self.n // world)
        nl += nl & 1
        self.c0, self.c1 = min(self.n, rank * nl), min(self.n, rank * nl + nl)
        self.nl = nl
        pl = -(-self.p // world)
        self.pl = pl
        self.x0, self.x1 = min(self.p, rank * pl), min(self.p, rank * pl + pl)
        self.method, self.theta, self.alpha = method, theta, alpha
        self.orc = O.oracle()
        self.rng = O.Rng()
        self.orc.rng_init(C.byref(self.rng), seed)
        self.a_sq = np.array([np.dot(r, r) for r in self.A])
        self.a_sq_g = self.allgather(self.a_sq)
        self.a_fro = float(np.sum(self.a_sq_g))
        self.cum = np.cumsum(self.a_sq_g)
        self.R = self.C - (self.A @ X0) @ B
        self.cyclic = 0

    # -- collectives
    def allgather(self, arr):
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).reshape(-1)
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t)
        return np.concatenate([o.numpy() for o in out])

    def allreduce(self, arr):
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).copy())
        dist.all_reduce(t)
        return t.numpy()

    def unit(self):
        return float(self.orc.rng_next_u64(C.byref(self.rng)) >> 11) * 2.0 ** -53

    # -- the grouped norms exchange + k_sel1's commit
    def records(self):
        r_sq = np.einsum("ij,ij->i", self.R, self.R)
        ratios = np.where(self.a_sq > 0, r_sq / np.where(self.a_sq > 0, self.a_sq, 1), -np.inf)
        j = int(np.argmax(ratios))  # first max = smallest index
        rec = np.array([float(np.sum(r_sq)), ratios[j], float(self.row0 + j)])
        # one grouped exchange: the ‖R_l‖² slice and the record of every shard
        both = self.allgather(np.concatenate([r_sq, rec])).reshape(self.world, self.ml + 3)
        self.r_sq_g = both[:, :self.ml].reshape(-1)
        recs = both[:, self.ml:]
        s, mx, ax = 0.0, -np.inf, None
        for r in range(self.world):  # rank order, smallest index on ties
            s += recs[r, 0]
            if recs[r, 1] > mx or (recs[r, 1] == mx and recs[r, 2] < ax):
                mx, ax = recs[r, 1], recs[r, 2]
        self.r_fro, self.max_ratio, self.argmax = s, mx, int(ax)

    # -- k_sel1's selection: every rank, over the GLOBAL rows, identically
    def select(self):
        if self.method == O.MWRBK:
            return self.argmax
        if self.method == O.BK:
            while True:
                i = self.cyclic
                self.cyclic = (self.cyclic + 1) % len(self.a_sq_g)
                if self.a_sq_g[i] > 0:
                    return i
        if self.method == O.RBK:
            t = self.unit() * self.cum[-1]
            lo = int(np.searchsorted(self.cum, t, side="right"))
            while lo > 0 and self.cum[lo] == self.cum[lo - 1]:
                lo -= 1
            return lo
        th = self.theta
        zeta = th * (self.max_ratio / self.r_fro) + (1.0 - th) / self.a_fro
        rows = np.arange(len(self.a_sq_g))
        member = (self.a_sq_g > 0) & ((rows == self.argmax) |
                                       (self.r_sq_g >= zeta * self.a_sq_g * self.r_fro))
        idx = np.nonzero(member)[0]
        cum = np.cumsum(self.r_sq_g[idx])  # ascending member order (solver.hpp:243-248)
        target = self.unit() * cum[-1]
        lo = int(np.searchsorted(cum, target, side="right"))  # upper_bound (rng.hpp:93)
        if lo >= len(cum):
            lo = len(cum) - 1
        while lo > 0 and cum[lo] == cum[lo - 1]:  # walk back over zero weights (:96-97)
            lo -= 1
        return int(idx[lo])

    def step(self):
        sel = self.select()  # the same row on every rank
        owner = sel // self.ml
        pack = np.zeros(self.n + self.p + 2)
        if owner == self.rank:
            il = sel - self.row0
            pack[:self.n] = self.R[il]
            pack[self.n:self.n + self.p] = self.A[il]
            pack[-2] = sel
            pack[-1] = self.alpha / self.a_sq[il]
        pack = self.allreduce(pack)
        Ri, Ai, i, coef = pack[:self.n], pack[self.n:self.n + self.p], int(pack[-2]), pack[-1]
        y = self.allreduce(self.B[:, self.c0:self.c1] @ Ri[self.c0:self.c1])
        zs = np.zeros(self.nl)
        zs[:self.c1 - self.c0] = y @ self.B[:, self.c0:self.c1]
        z = self.allgather(zs)[:self.n]
        self.X[self.x0:self.x1] += (coef * Ai[self.x0:self.x1])[:, None] * y[None, :]
        g = self.A @ Ai
        self.R -= (coef * g)[:, None] * z[None, :]
        self.records()
        return i

    def gather_X(self):
        pad = np.zeros((self.pl, self.X.shape[1]))
        pad[:self.x1 - self.x0] = self.X[self.x0:self.x1]
        return self.allgather(pad).reshape(self.world * self.pl, -1)[:self.p]
