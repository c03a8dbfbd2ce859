"""Python mirror of the reference's solver API (solver.hpp:16-532) over the C-ABI.

Names, argument meaning and error behaviour follow ``axb::`` so the parity tests
read like the reference's own tests (proj/tests/test_solver.cpp):

    Method.bk()/rbk()/grbk()/rgrbk(θ)/mwrbk()     solver.hpp:20-62
    AlphaRule.Safe/Paper/Fixed                     :68
    StopRule.solution_rrn(tol, X_ref) / residual_rel(tol)   :79-98
    SolveConfig, TracePoint, SolveReport, Terminated        :100-133
    Solver(A, B, C, X0, cfg).step()/run()/update_row()/...  :143-515
    solve(A, B, C, X0, cfg)                                  :518-532

Every call goes to libaxb_b200.so (hand-written sm_100a CUDA); there is no CPU path.
Inputs may be host numpy arrays or device tensors (anything exposing
``__cuda_array_interface__`` or a torch CUDA tensor), float64, row-major.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .errors import ConfigError, DivergenceError, raise_status

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class MethodTag(enum.IntEnum):  # solver.hpp:16
    BK = 0
    RBK = 1
    GRBK = 2
    RGRBK = 3
    MWRBK = 4


@dataclass
class Method:  # solver.hpp:20-62
    tag: MethodTag = MethodTag.RBK
    theta: Optional[float] = None

    @staticmethod
    def bk():
        return Method(MethodTag.BK)

    @staticmethod
    def rbk():
        return Method(MethodTag.RBK)

    @staticmethod
    def grbk():
        return Method(MethodTag.GRBK)

    @staticmethod
    def rgrbk(theta: float):
        return Method(MethodTag.RGRBK, theta)

    @staticmethod
    def mwrbk():
        return Method(MethodTag.MWRBK)

    def validate(self):
        if self.tag == MethodTag.RGRBK:
            if self.theta is None:
                raise ConfigError("rgrbk requires theta")
            if not (0.0 < self.theta < 1.0):
                raise ConfigError("theta must lie strictly in (0, 1)")
        elif self.theta is not None:
            raise ConfigError("theta is only valid for rgrbk")

    def label(self) -> str:
        return self.tag.name.lower()

    @staticmethod
    def parse(name: str, theta: Optional[float] = None):
        table = {"bk": Method.bk, "rbk": Method.rbk, "grbk": Method.grbk, "mwrbk": Method.mwrbk}
        if name in table:
            return table[name]()
        if name == "rgrbk":
            if theta is None:
                raise ConfigError("rgrbk requires theta")
            return Method.rgrbk(theta)
        raise ConfigError(f"unknown method '{name}'")


class AlphaRule(enum.IntEnum):  # solver.hpp:68
    Safe = 0
    Paper = 1
    Fixed = 2


@dataclass
class StopRule:  # solver.hpp:79-98
    class Kind(enum.IntEnum):
        SolutionRrn = 0
        ResidualRel = 1

    kind: "StopRule.Kind" = Kind.ResidualRel
    tol: float = 1e-6
    reference: object = None

    @staticmethod
    def solution_rrn(tol, reference):
        return StopRule(StopRule.Kind.SolutionRrn, tol, reference)

    @staticmethod
    def residual_rel(tol):
        return StopRule(StopRule.Kind.ResidualRel, tol, None)


@dataclass
class SolveConfig:  # solver.hpp:100-109
    method: Method = field(default_factory=Method.rbk)
    alpha_rule: AlphaRule = AlphaRule.Safe
    alpha_value: float = 0.0
    stop: StopRule = field(default_factory=lambda: StopRule.residual_rel(1e-6))
    max_iter: int = 200000
    seed: int = 0
    record_trace: bool = False
    refresh_interval: int = 1000


@dataclass
class TracePoint:  # solver.hpp:111-116
    k: int
    rrn: float
    residual_rel: float
    selected_row: int


class Terminated(enum.IntEnum):  # solver.hpp:118
    Tolerance = 0
    MaxIter = 1


@dataclass
class SolveReport:  # solver.hpp:120-133
    iterations: int = 0
    wall_seconds: float = 0.0
    final_rrn: float = 0.0
    final_residual_rel: float = 0.0
    terminated_by: Terminated = Terminated.MaxIter
    trace: List[TracePoint] = field(default_factory=list)
    X: Optional[np.ndarray] = None
    alpha: float = 0.0
    seed: int = 0
    method_label: str = ""
    alpha_outside_bound: bool = False
    skipped_zero_rows: int = 0


def trace_point_due(k: int) -> bool:  # solver.hpp:136
    return k < 10000 or k % 10 == 0


kDriftGuardScale = 1e-8  # solver.hpp:138


@dataclass
class Options:
    """B200 execution options (axb_options; no reference analogue)."""

    device: int = 0
    cache_gram: int = -1          # -1 auto, 0 GEMV g = A·A_iᵀ per step, 1 cache G = A·Aᵀ
    spectral_on_device: int = -1  # -1 auto, 0 host (bitwise reference α), 1 device
    graph_iters: int = 0          # iterations per captured CUDA graph (0 = default)
    tie_guard: int = 1            # sequential re-check of near-boundary greedy draws (2: always)
    spectral_max_iter: int = 0    # 0 = reference default 5000
    alpha_override: float = 0.0   # >0: use verbatim (e.g. the oracle's α)
    # row sharding: this solver owns rows [row_offset, row_offset+m)
    # of an m_global-row system; nccl_comm from nccl_comm_create() (see shard.py)
    nccl_comm: int = 0
    world_size: int = 1
    rank: int = 0
    m_global: int = 0
    row_offset: int = 0
    # SMs the persistent kernel of this handle may occupy (0 = all): handles that
    # run concurrently from their own host threads share one GPU
    sm_share: int = 0


def _device_ptr(a):
    """Device pointer of a CUDA array (torch tensor or __cuda_array_interface__), else None."""
    if hasattr(a, "__cuda_array_interface__"):
        iface = a.__cuda_array_interface__
        if iface.get("typestr") not in ("<f8", "f8"):
            raise ConfigError("device inputs must be float64")
        if iface.get("strides") not in (None,) and not _contig(iface):
            raise ConfigError("device inputs must be C-contiguous")
        return iface["data"][0]
    return None


def _contig(iface):
    shape, strides = iface["shape"], iface["strides"]
    if strides is None:
        return True
    expect = 8
    for dim, st in zip(reversed(shape), reversed(strides)):
        if dim > 1 and st != expect:
            return False
        expect *= dim
    return True


def _is_csr(a):
    return hasattr(a, "indptr") and hasattr(a, "indices") and hasattr(a, "format")


def _shape(a):
    if _is_csr(a):
        return tuple(a.shape)
    if hasattr(a, "__cuda_array_interface__"):
        return tuple(a.__cuda_array_interface__["shape"])
    return tuple(np.shape(a))


class Solver:
    """axb::Solver<DenseMatrix,DenseMatrix> (solver.hpp:143-515) on a B200."""

    def __init__(self, A, B, C_, X0, cfg: SolveConfig, options: Optional[Options] = None):
        lib = _lib.load()
        self._lib = lib
        self._h = None
        cfg.method.validate()
        opts = options or Options()
        m, p = _shape(A)
        q, n = _shape(B)
        if X0 is not None and _shape(X0) != (p, q):
            from .errors import ShapeError
            raise ShapeError(f"solve: X0 must be {p}x{q}")
        if _shape(C_) != (m, n):
            from .errors import ShapeError
            raise ShapeError(f"solve: C must be {m}x{n}")
        # checked before any buffer is handed to the library (solver.hpp:182-185)
        if cfg.stop.kind == StopRule.Kind.SolutionRrn and cfg.stop.reference is not None:
            if _shape(cfg.stop.reference) != (p, q):
                from .errors import ShapeError
                raise ShapeError("reference solution shape mismatch")
        self.m, self.p, self.q, self.n = m, p, q, n
        on_dev = _device_ptr(A) is not None
        keep = []

        def ptr(a):
            if a is None:
                return None
            if on_dev:
                d = _device_ptr(a)
                if d is None:
                    raise ConfigError("mix of host and device inputs")
                return d
            arr = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(arr)
            return arr.ctypes.data

        c = _lib.AxbConfig()
        c.method = int(cfg.method.tag)
        c.has_theta = 0 if cfg.method.theta is None else 1
        c.theta = 0.0 if cfg.method.theta is None else float(cfg.method.theta)
        c.alpha_rule = int(cfg.alpha_rule)
        c.stop_kind = int(cfg.stop.kind)
        c.alpha_value = float(cfg.alpha_value)
        c.tol = float(cfg.stop.tol)
        c.reference = ptr(cfg.stop.reference) if cfg.stop.reference is not None else None
        c.max_iter = int(cfg.max_iter)
        c.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
        c.record_trace = 1 if cfg.record_trace else 0
        c.refresh_interval = int(cfg.refresh_interval)
        o = _lib.AxbOptions()
        lib.axb_options_default(C.byref(o))
        o.device = opts.device
        o.inputs_on_device = 1 if on_dev else 0
        o.cache_gram = opts.cache_gram
        o.spectral_on_device = opts.spectral_on_device
        o.graph_iters = opts.graph_iters
        o.tie_guard = 2 if opts.tie_guard == 2 else (1 if opts.tie_guard else 0)
        o.spectral_max_iter = opts.spectral_max_iter
        o.alpha_override = opts.alpha_override
        o.nccl_comm = opts.nccl_comm or None
        o.world_size = opts.world_size
        o.rank = opts.rank
        o.m_global = opts.m_global
        o.row_offset = opts.row_offset
        o.sm_share = opts.sm_share
        h = C.c_void_p()
        if _is_csr(A) or _is_csr(B):
            if on_dev:
                raise ConfigError("CSR operands are host arrays")

            def desc(M):
                d = _lib.AxbMatrix()
                d.rows, d.cols = M.shape
                if _is_csr(M):
                    M = M.tocsr()
                    M.sort_indices()
                    rp = np.ascontiguousarray(M.indptr, dtype=np.uint64)
                    ci = np.ascontiguousarray(M.indices, dtype=np.uint64)
                    vv = np.ascontiguousarray(M.data, dtype=np.float64)
                    keep.extend([rp, ci, vv])
                    d.kind, d.nnz = 1, vv.size
                    d.row_ptr, d.col_idx, d.values = rp.ctypes.data, ci.ctypes.data, vv.ctypes.data
                else:
                    d.kind = 0
                    d.dense = ptr(M)
                return d

            dA, dB = desc(A), desc(B)
            st = lib.axb_solver_create_ex(C.byref(dA), C.byref(dB), ptr(C_), ptr(X0), C.byref(c),
                                          C.byref(o), C.byref(h))
        else:
            st = lib.axb_solver_create(ptr(A), m, p, ptr(B), q, n, ptr(C_), ptr(X0), C.byref(c),
                                       C.byref(o), C.byref(h))
        if st:
            raise_status(st, lib.axb_last_create_error().decode())
        self._h = h
        self.cfg = cfg

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.axb_solver_destroy(self._h)
            self._h = None

    def _chk(self, st, **kw):
        if st:
            if not kw:
                k = C.c_uint64(); v = C.c_double()
                self._lib.axb_solver_last_error_info(self._h, C.byref(k), C.byref(v))
                kw = {"iteration": k.value, "residual_norm": v.value}
            raise_status(st, self._lib.axb_solver_last_error(self._h).decode(), **kw)

    # -- selection rules (solver.hpp:197-258) --
    def select_cyclic(self):
        r = C.c_uint64(); self._chk(self._lib.axb_solver_select_cyclic(self._h, C.byref(r))); return r.value

    def select_rbk(self):
        r = C.c_uint64(); self._chk(self._lib.axb_solver_select_rbk(self._h, C.byref(r))); return r.value

    def select_greedy(self, theta):
        r = C.c_uint64()
        self._chk(self._lib.axb_solver_select_greedy(self._h, theta, C.byref(r)))
        return r.value

    def select_grbk(self):
        return self.select_greedy(0.5)

    def select_mwrbk(self):
        r = C.c_uint64(); self._chk(self._lib.axb_solver_select_mwrbk(self._h, C.byref(r))); return r.value

    def greedy_threshold(self, theta):
        v = C.c_double(); self._chk(self._lib.axb_solver_greedy_threshold(self._h, theta, C.byref(v))); return v.value

    def grbk_threshold(self):
        return self.greedy_threshold(0.5)

    def rgrbk_threshold(self, theta):
        v = C.c_double(); self._chk(self._lib.axb_solver_rgrbk_threshold(self._h, theta, C.byref(v))); return v.value

    def greedy_index_set(self, theta):
        out = np.empty(self.m, dtype=np.uint64)
        cnt = C.c_uint64()
        self._chk(self._lib.axb_solver_greedy_index_set(self._h, theta, out.ctypes.data_as(_u64p), C.byref(cnt)))
        return [int(v) for v in out[: cnt.value]]

    def max_residual_ratio(self):
        r = C.c_uint64(); v = C.c_double()
        self._chk(self._lib.axb_solver_max_residual_ratio(self._h, C.byref(r), C.byref(v)))
        return r.value, v.value

    # -- kernel / loop (solver.hpp:264-372) --
    def update_row(self, i):
        self._chk(self._lib.axb_solver_update_row(self._h, int(i)))

    def step(self):
        r = C.c_uint64()
        self._chk(self._lib.axb_solver_step(self._h, C.byref(r)))
        return r.value

    def steps(self, k, mirror_refresh=False):
        """k step() calls batched on the device; returns the selected rows."""
        rows = np.empty(max(int(k), 1), dtype=np.uint64)
        self._chk(self._lib.axb_solver_steps(self._h, int(k), rows.ctypes.data_as(_u64p),
                                             1 if mirror_refresh else 0))
        return rows[: int(k)]

    def replay(self, rows, mirror_refresh=False):
        """Iterate on a given index stream (e.g. the reference's trace)."""
        r = np.ascontiguousarray(rows, dtype=np.uint64)
        self._chk(self._lib.axb_solver_replay(self._h, int(r.size), r.ctypes.data_as(_u64p),
                                              1 if mirror_refresh else 0))

    def run(self) -> SolveReport:
        cap = 0
        if self.cfg.record_trace:
            mi = int(self.cfg.max_iter)
            cap = mi if mi <= 10000 else 10000 + (mi - 10000) // 10 + 1
        tk = np.zeros(max(cap, 1), dtype=np.uint64)
        trr = np.zeros(max(cap, 1))
        trl = np.zeros(max(cap, 1))
        trw = np.zeros(max(cap, 1), dtype=np.uint64)
        X = np.empty((self.p, self.q))
        rep = _lib.AxbReport()
        st = self._lib.axb_solver_run(self._h, C.byref(rep), tk.ctypes.data_as(_u64p),
                                      trr.ctypes.data_as(_dp), trl.ctypes.data_as(_dp),
                                      trw.ctypes.data_as(_u64p), cap, X.ctypes.data_as(_dp))
        self._chk(st, iteration=rep.diverged_iteration, residual_norm=rep.diverged_residual)
        n = min(rep.trace_len, cap)
        return SolveReport(
            iterations=rep.iterations, wall_seconds=rep.wall_seconds, final_rrn=rep.final_rrn,
            final_residual_rel=rep.final_residual_rel, terminated_by=Terminated(rep.terminated_by),
            trace=[TracePoint(int(tk[t]), float(trr[t]), float(trl[t]), int(trw[t])) for t in range(n)],
            X=X, alpha=rep.alpha, seed=rep.seed, method_label=self.cfg.method.label(),
            alpha_outside_bound=bool(rep.alpha_outside_bound), skipped_zero_rows=rep.skipped_zero_rows)

    def _report(self, rep, X, trace=()):
        return SolveReport(
            iterations=rep.iterations, wall_seconds=rep.wall_seconds, final_rrn=rep.final_rrn,
            final_residual_rel=rep.final_residual_rel, terminated_by=Terminated(rep.terminated_by),
            trace=list(trace), X=X, alpha=rep.alpha, seed=rep.seed,
            method_label=self.cfg.method.label(),
            alpha_outside_bound=bool(rep.alpha_outside_bound),
            skipped_zero_rows=rep.skipped_zero_rows)

    # -- accessors (solver.hpp:376-436) --
    def iteration(self):
        return int(self._lib.axb_solver_iteration(self._h))

    def alpha(self):
        return self._lib.axb_solver_alpha(self._h)

    def spectral_norm_b(self):
        return self._lib.axb_solver_spectral_norm_b(self._h)

    def alpha_outside_bound(self):
        return bool(self._lib.axb_solver_alpha_outside_bound(self._h))

    def gram_cached(self):
        """True when G = A·Aᵀ is cached; False when g = A·A_iᵀ is formed per step."""
        return bool(self._lib.axb_solver_gram_cached(self._h))

    def _vec(self, fn, shape):
        out = np.empty(shape)
        self._chk(fn(self._h, out.ctypes.data_as(_dp)))
        return out

    def X(self):
        return self._vec(self._lib.axb_solver_get_X, (self.p, self.q))

    def R(self):
        return self._vec(self._lib.axb_solver_get_R, (self.m, self.n))

    def residual_row_sq(self):
        return self._vec(self._lib.axb_solver_get_r_sq, (self.m,))

    def a_row_sq(self):
        return self._vec(self._lib.axb_solver_get_a_sq, (self.m,))

    def a_fro_sq(self):
        return self._lib.axb_solver_a_fro_sq(self._h)

    def _scalar(self, fn):
        v = C.c_double()
        self._chk(fn(self._h, C.byref(v)))
        return v.value

    def residual_fro_sq(self):
        return self._scalar(self._lib.axb_solver_residual_fro_sq)

    def current_metric(self):
        return self._scalar(self._lib.axb_solver_current_metric)

    def current_residual_rel(self):
        return self._scalar(self._lib.axb_solver_current_residual_rel)

    def exact_metric(self):
        return self._scalar(self._lib.axb_solver_exact_metric)

    def exact_residual_rel(self):
        return self._scalar(self._lib.axb_solver_exact_residual_rel)

    def residual_drift(self):
        return self._scalar(self._lib.axb_solver_residual_drift)

    def checkpoint(self):
        self._chk(self._lib.axb_solver_checkpoint(self._h))

    # -- measurement hooks --
    def set_profiling(self, on: bool):
        self._lib.axb_solver_set_profiling(self._h, 1 if on else 0)

    def kernel_times(self):
        """Average in-pipeline ms per launch of K4 (y), K4b+K5 (z, X), K2 (profiled runs)."""
        out = (C.c_double * 3)()
        self._lib.axb_solver_kernel_times(self._h, out)
        return {"yg_ms": out[0], "zx_ms": out[1], "k2_ms": out[2]}

    def collective_times(self):
        """Row-sharded solvers, profiled runs: average ms per iteration of each
        exchange step (zeros on one GPU)."""
        out = (C.c_double * 5)()
        self._lib.axb_solver_collective_times(self._h, out)
        return {"y_allreduce_ms": out[0], "z_allgather_ms": out[1],
                "norms_allgather_ms": out[2], "select_kernels_ms": out[3],
                "row_allreduce_ms": out[4]}

    def selection_stats(self):
        """Greedy draws made on the device and how many of them took the exact
        sequential walk of the reference (the tie guard's fallback)."""
        d = (C.c_uint64 * 8)()
        self._chk(self._lib.axb_solver_debug_state(self._h, d))
        return {"greedy_selections": int(d[5]), "sequential_walks": int(d[6])}

    def last_timing(self):
        a = C.c_double(); b = C.c_double(); c = C.c_uint64(); d = C.c_uint64()
        self._lib.axb_solver_last_timing(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d))
        return {"loop_ms": a.value, "k2_ms": b.value, "k2_launches": c.value,
                "kernel_launches": d.value}


def run_many(solvers: List["Solver"], return_exceptions: bool = False) -> list:
    """run() on many independent solvers of one device in one batch
    (axb_solvers_run): small systems advance together, one CTA each, through a
    single launch per refresh segment.  Each result equals that
    solver's own run(), without the trace.  A failed solve raises its
    reference exception — or, with return_exceptions, is returned in its slot."""
    if not solvers:
        return []
    lib = _lib.load()
    k = len(solvers)
    hs = (C.c_void_p * k)(*[s._h for s in solvers])
    reps = (_lib.AxbReport * k)()
    xs = [np.empty((s.p, s.q)) for s in solvers]
    xp = (_dp * k)(*[x.ctypes.data_as(_dp) for x in xs])
    sts = (C.c_int32 * k)()
    st = lib.axb_solvers_run(hs, k, reps, xp, sts)
    if st:
        raise_status(st, lib.axb_last_create_error().decode())
    out = []
    for i, s in enumerate(solvers):
        if sts[i]:
            try:
                s._chk(sts[i], iteration=reps[i].diverged_iteration,
                       residual_norm=reps[i].diverged_residual)
            except Exception as e:  # noqa: BLE001
                if not return_exceptions:
                    raise
                out.append(e)
            continue
        out.append(s._report(reps[i], xs[i]))
    return out


def solve(A, B, C_, X0, cfg: SolveConfig, options: Optional[Options] = None) -> SolveReport:
    """axb::solve (solver.hpp:518-532)."""
    return Solver(A, B, C_, X0, cfg, options).run()
