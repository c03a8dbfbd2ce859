"""ctypes bindings for the CPU ORACLE (test infrastructure only).

Two libraries with the same shape of API:

* ``oracle/liboracle.so``       — the plain-C restatement (``oracle/axb_oracle.c``);
* ``oracle/_ref/libaxbref.so``  — the UNMODIFIED reference engine compiled from
  ``/root/reference/proj/include`` (``oracle/ref_driver.cpp``); present only
  where it was built (this container, and GPU boxes that received the prebuilt .so).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs import
this module.  The product (``paper_2408_05444_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "liboracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libaxbref.so")

BK, RBK, GRBK, RGRBK, MWRBK = range(5)
SAFE, PAPER, FIXED = range(3)
SOLUTION_RRN, RESIDUAL_REL = range(2)

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


class Config(C.Structure):
    """SolveConfig (solver.hpp:100-109) — same layout as axb_config / orc_config."""

    _fields_ = [
        ("method", C.c_int32),
        ("has_theta", C.c_int32),
        ("theta", C.c_double),
        ("alpha_rule", C.c_int32),
        ("stop_kind", C.c_int32),
        ("alpha_value", C.c_double),
        ("tol", C.c_double),
        ("reference", _dp),
        ("max_iter", C.c_uint64),
        ("seed", C.c_uint64),
        ("record_trace", C.c_int32),
        ("_pad", C.c_int32),
        ("refresh_interval", C.c_uint64),
    ]


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_uint64),
        ("wall_seconds", C.c_double),
        ("final_rrn", C.c_double),
        ("final_residual_rel", C.c_double),
        ("terminated_by", C.c_int32),
        ("alpha_outside_bound", C.c_int32),
        ("alpha", C.c_double),
        ("seed", C.c_uint64),
        ("skipped_zero_rows", C.c_uint64),
        ("trace_len", C.c_uint64),
        ("diverged_iteration", C.c_uint64),
        ("diverged_residual", C.c_double),
    ]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def make_config(method=GRBK, theta=None, alpha_rule=SAFE, alpha_value=0.0, stop_kind=RESIDUAL_REL,
                tol=1e-6, reference=None, max_iter=200000, seed=0, record_trace=False,
                refresh_interval=1000):
    cfg = Config()
    cfg.method = method
    cfg.has_theta = 0 if theta is None else 1
    cfg.theta = 0.0 if theta is None else float(theta)
    cfg.alpha_rule = alpha_rule
    cfg.alpha_value = alpha_value
    cfg.stop_kind = stop_kind
    cfg.tol = tol
    keep = None
    if reference is not None:
        keep = np.ascontiguousarray(reference, dtype=np.float64)
        cfg.reference = keep.ctypes.data_as(_dp)
    cfg.max_iter = max_iter
    cfg.seed = seed
    cfg.record_trace = 1 if record_trace else 0
    cfg.refresh_interval = refresh_interval
    cfg._keep = keep  # keep the reference buffer alive as long as the config
    return cfg


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_dp)


def ensure_built():
    """Compile liboracle.so (and _ref where /root/reference exists)."""
    if not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(ORACLE_DIR, "axb_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


class _Lib:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        self._declare()

    def _f(self, name, restype, argtypes):
        fn = getattr(self.lib, self.prefix + name)
        fn.restype = restype
        fn.argtypes = argtypes
        return fn


class OracleLib(_Lib):
    """The C restatement (oracle/axb_oracle.c)."""

    prefix = "orc_"

    def _declare(self):
        S = C.c_size_t
        self.generate_gaussian = self._f(
            "generate_gaussian", None, [C.c_uint64, S, S, S, S, _dp, _dp, _dp, _dp])
        self.spectral_norm = self._f(
            "spectral_norm", C.c_double, [_dp, S, S, C.c_double, S, C.POINTER(C.c_int), _dp])
        self.create = self._f(
            "solver_create", C.c_void_p,
            [_dp, S, S, _dp, S, S, _dp, _dp, C.POINTER(Config), C.POINTER(C.c_int), C.c_char_p, S])
        self.destroy = self._f("solver_destroy", None, [C.c_void_p])
        self.last_error = self._f("solver_last_error", C.c_char_p, [C.c_void_p])
        self.step = self._f("solver_step", C.c_int, [C.c_void_p, _u64p])
        self.update_row = self._f("solver_update_row", C.c_int, [C.c_void_p, C.c_uint64])
        self.run = self._f("solver_run", C.c_int,
                           [C.c_void_p, C.POINTER(Report), _u64p, _dp, _dp, _u64p, C.c_uint64, _dp])
        self.checkpoint = self._f("solver_checkpoint", C.c_int, [C.c_void_p])
        self.greedy_threshold = self._f("solver_greedy_threshold", C.c_int,
                                        [C.c_void_p, C.c_double, _dp])
        self.rgrbk_threshold = self._f("solver_rgrbk_threshold", C.c_int,
                                       [C.c_void_p, C.c_double, _dp])
        self.greedy_index_set = self._f("solver_greedy_index_set", C.c_int,
                                        [C.c_void_p, C.c_double, _u64p, _u64p])
        self.max_residual_ratio = self._f("solver_max_residual_ratio", C.c_int,
                                          [C.c_void_p, _u64p, _dp])
        self.select_cyclic = self._f("solver_select_cyclic", C.c_int, [C.c_void_p, _u64p])
        self.select_rbk = self._f("solver_select_rbk", C.c_int, [C.c_void_p, _u64p])
        self.select_greedy = self._f("solver_select_greedy", C.c_int,
                                     [C.c_void_p, C.c_double, _u64p])
        self.select_mwrbk = self._f("solver_select_mwrbk", C.c_int, [C.c_void_p, _u64p])
        self.exact_metric = self._f("solver_exact_metric", C.c_int, [C.c_void_p, _dp])
        self.residual_drift = self._f("solver_residual_drift", C.c_int, [C.c_void_p, _dp])
        self.current_metric = self._f("solver_current_metric", C.c_double, [C.c_void_p])
        self.iteration = self._f("solver_iteration", C.c_uint64, [C.c_void_p])
        self.alpha = self._f("solver_alpha", C.c_double, [C.c_void_p])
        self.spectral_norm_b = self._f("solver_spectral_norm_b", C.c_double, [C.c_void_p])
        self.a_fro_sq = self._f("solver_a_fro_sq", C.c_double, [C.c_void_p])
        self.residual_fro_sq = self._f("solver_residual_fro_sq", C.c_double, [C.c_void_p])
        self.get_X = self._f("solver_get_X", None, [C.c_void_p, _dp])
        self.get_R = self._f("solver_get_R", None, [C.c_void_p, _dp])
        self.get_r_sq = self._f("solver_get_r_sq", None, [C.c_void_p, _dp])
        self.get_a_sq = self._f("solver_get_a_sq", None, [C.c_void_p, _dp])
        self.rng_state = self._f("solver_rng_state", None, [C.c_void_p, _u64p])
        self.rng_init = self._f("rng_init", None, [C.c_void_p, C.c_uint64])
        self.rng_next_u64 = self._f("rng_next_u64", C.c_uint64, [C.c_void_p])
        self.rng_gauss = self._f("rng_gauss", C.c_double, [C.c_void_p])
        self.rng_substream = self._f("rng_substream", None, [C.c_void_p, C.c_uint64, C.c_void_p])
        self.rng_categorical_cdf = self._f("rng_categorical_cdf", C.c_size_t,
                                           [C.c_void_p, _dp, C.c_size_t, C.POINTER(C.c_int)])
        self.create_prepared = self._f(
            "solver_create_prepared", C.c_void_p,
            [_dp, S, S, _dp, S, S, _dp, _dp, _dp, _dp, _dp, C.c_double, C.POINTER(Config),
             C.POINTER(C.c_int)])
        self.steps_c = self._f("solver_steps", C.c_int, [C.c_void_p, C.c_uint64, _u64p])


class RefLib(_Lib):
    """The unmodified reference engine (oracle/_ref/libaxbref.so)."""

    prefix = "ref_"

    def _declare(self):
        S = C.c_size_t
        self.generate_gaussian = self._f(
            "generate_gaussian", None, [C.c_uint64, S, S, S, S, _dp, _dp, _dp, _dp])
        self.rng_stream = self._f("rng_stream", C.c_uint64, [C.c_uint64, C.c_uint64, _u64p, _dp])
        self.substream_seed = self._f("substream_seed", C.c_uint64, [C.c_uint64, C.c_uint64])
        self.spectral_norm = self._f("spectral_norm", C.c_double,
                                     [_dp, S, S, C.c_double, C.c_uint64, C.POINTER(C.c_int)])
        self.create = self._f("solver_create", C.c_void_p,
                              [_dp, S, S, _dp, S, S, _dp, _dp, C.POINTER(Config), C.POINTER(C.c_int)])
        self.destroy = self._f("solver_destroy", None, [C.c_void_p])
        self.last_error = self._f("solver_last_error", C.c_char_p, [C.c_void_p])
        self.step = self._f("solver_step", C.c_int, [C.c_void_p, _u64p])
        self.steps = self._f("solver_steps", C.c_int,
                             [C.c_void_p, C.c_uint64, _u64p, C.c_int, C.c_uint64])
        self.update_row = self._f("solver_update_row", C.c_int, [C.c_void_p, C.c_uint64])
        self.run = self._f("solver_run", C.c_int,
                           [C.c_void_p, C.POINTER(Report), _u64p, _dp, C.c_uint64, _dp])
        self.checkpoint = self._f("solver_checkpoint", C.c_int, [C.c_void_p])
        self.greedy_threshold = self._f("solver_greedy_threshold", C.c_int,
                                        [C.c_void_p, C.c_double, _dp])
        self.greedy_index_set = self._f("solver_greedy_index_set", C.c_int,
                                        [C.c_void_p, C.c_double, _u64p, _u64p])
        self.max_residual_ratio = self._f("solver_max_residual_ratio", C.c_int,
                                          [C.c_void_p, _u64p, _dp])
        self.exact_metric = self._f("solver_exact_metric", C.c_int, [C.c_void_p, _dp])
        self.residual_drift = self._f("solver_residual_drift", C.c_int, [C.c_void_p, _dp])
        self.current_metric = self._f("solver_current_metric", C.c_double, [C.c_void_p])
        self.iteration = self._f("solver_iteration", C.c_uint64, [C.c_void_p])
        self.alpha = self._f("solver_alpha", C.c_double, [C.c_void_p])
        self.spectral_norm_b = self._f("solver_spectral_norm_b", C.c_double, [C.c_void_p])
        self.a_fro_sq = self._f("solver_a_fro_sq", C.c_double, [C.c_void_p])
        self.residual_fro_sq = self._f("solver_residual_fro_sq", C.c_double, [C.c_void_p])
        self.get_X = self._f("solver_get_X", None, [C.c_void_p, _dp])
        self.get_R = self._f("solver_get_R", None, [C.c_void_p, _dp])
        self.get_r_sq = self._f("solver_get_r_sq", None, [C.c_void_p, _dp])
        self.get_a_sq = self._f("solver_get_a_sq", None, [C.c_void_p, _dp])
        self.blur_operator = self._f("blur_operator", C.c_uint64,
                                     [S, S, S, C.c_double, _u64p, _u64p, _dp])
        self.synthetic_stack = self._f("synthetic_stack", None, [S, S, _dp, _dp])
        self.sparse_steps_c = self._f(
            "sparse_steps", C.c_int,
            [_u64p, _u64p, _dp, S, S, _u64p, _u64p, _dp, _dp, S, S, _dp, _dp,
             C.POINTER(Config), C.c_uint64, _u64p, _dp, _dp, _dp, C.c_char_p])

    def blur_model(self, h, w, ksize, sigma):
        """imaging.hpp:93-136 + :276-310: (A as scipy CSR h·w × h·w, X* stack
        (h·w)×3, A_c 3×3)."""
        import scipy.sparse as sp

        nnz = self.blur_operator(h, w, ksize, sigma, None, None, None)
        rp = np.empty(h * w + 1, dtype=np.uint64)
        ci = np.empty(nnz, dtype=np.uint64)
        v = np.empty(nnz)
        self.blur_operator(h, w, ksize, sigma, rp.ctypes.data_as(_u64p), ci.ctypes.data_as(_u64p),
                           _ptr(v))
        A = sp.csr_matrix((v, ci.astype(np.int64), rp.astype(np.int64)), shape=(h * w, h * w))
        X = np.empty((h * w, 3))
        Ac = np.empty((3, 3))
        self.synthetic_stack(h, w, _ptr(X), _ptr(Ac))
        return A, X, Ac

    def sparse_steps(self, A, B, Cm, X0, cfg, k):
        """Solver<SparseMatrix, BMat> (B CSR or dense), k step() calls:
        rows, X, r_sq, α."""
        def parts(M):
            M = M.tocsr()
            M.sort_indices()
            return (np.ascontiguousarray(M.indptr, dtype=np.uint64),
                    np.ascontiguousarray(M.indices, dtype=np.uint64),
                    np.ascontiguousarray(M.data, dtype=np.float64))

        a = parts(A)
        m, p = A.shape
        q, n = B.shape
        bcsr = hasattr(B, "indptr")
        b = parts(B) if bcsr else None
        Bd = None if bcsr else np.ascontiguousarray(B, dtype=np.float64)
        Cm = np.ascontiguousarray(Cm, dtype=np.float64)
        X0 = np.zeros((p, q)) if X0 is None else np.ascontiguousarray(X0, dtype=np.float64)
        rows = np.empty(max(k, 1), dtype=np.uint64)
        X = np.empty((p, q))
        rs = np.empty(m)
        al = C.c_double()
        err = C.create_string_buffer(256)
        u = lambda t: t.ctypes.data_as(_u64p)  # noqa: E731
        code = self.sparse_steps_c(u(a[0]), u(a[1]), _ptr(a[2]), m, p,
                                   u(b[0]) if b else None, u(b[1]) if b else None,
                                   _ptr(b[2]) if b else None, _ptr(Bd), q, n, _ptr(Cm), _ptr(X0),
                                   C.byref(cfg), k, u(rows), _ptr(X), _ptr(rs), C.byref(al), err)
        if code:
            raise OracleError(code, err.value.decode())
        return rows[:k], X, rs, al.value


_oracle = None
_ref = None


def oracle() -> OracleLib:
    global _oracle
    if _oracle is None:
        ensure_built()
        _oracle = OracleLib(ORACLE_SO)
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> RefLib:
    global _ref
    if _ref is None:
        _ref = RefLib(REF_SO)
    return _ref


def generate(lib, seed, m, p, q, n):
    """problems.hpp:345-364 for Gaussian sources: returns A, B, X*, C."""
    A = np.empty((m, p)); B = np.empty((q, n)); X = np.empty((p, q)); Cm = np.empty((m, n))
    lib.generate_gaussian(seed, m, p, q, n, _ptr(A), _ptr(B), _ptr(X), _ptr(Cm))
    return A, B, X, Cm


class Solver:
    """Thin Python handle over either library's solver (mirrors axb::Solver)."""

    def __init__(self, lib, A, B, Cm, X0, cfg):
        self.lib = lib
        self.A = np.ascontiguousarray(A, dtype=np.float64)
        self.B = np.ascontiguousarray(B, dtype=np.float64)
        self.C = np.ascontiguousarray(Cm, dtype=np.float64)
        self.m, self.p = self.A.shape
        self.q, self.n = self.B.shape
        self.X0 = (np.zeros((self.p, self.q)) if X0 is None
                   else np.ascontiguousarray(X0, dtype=np.float64))
        self.cfg = cfg
        st = C.c_int(0)
        if isinstance(lib, OracleLib):
            buf = C.create_string_buffer(256)
            self.h = lib.create(_ptr(self.A), self.m, self.p, _ptr(self.B), self.q, self.n,
                                _ptr(self.C), _ptr(self.X0), C.byref(cfg), C.byref(st), buf, 256)
            msg = buf.value.decode()
        else:
            self.h = lib.create(_ptr(self.A), self.m, self.p, _ptr(self.B), self.q, self.n,
                                _ptr(self.C), _ptr(self.X0), C.byref(cfg), C.byref(st))
            msg = "reference ctor failed"
        if not self.h:
            raise OracleError(st.value, msg)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.destroy(self.h)
            self.h = None

    def _chk(self, code):
        if code:
            raise OracleError(code, self.lib.last_error(self.h).decode())

    def step(self):
        r = C.c_uint64()
        self._chk(self.lib.step(self.h, C.byref(r)))
        return r.value

    def steps(self, k, mirror_refresh=False, refresh_interval=0):
        rows = np.empty(k, dtype=np.uint64)
        if isinstance(self.lib, RefLib):
            self._chk(self.lib.steps(self.h, k, rows.ctypes.data_as(_u64p), int(mirror_refresh),
                                     refresh_interval))
        else:
            for t in range(k):
                rows[t] = self.step()
                if mirror_refresh and refresh_interval and self.iteration % refresh_interval == 0:
                    self.checkpoint()
        return rows

    def update_row(self, i):
        self._chk(self.lib.update_row(self.h, i))

    def checkpoint(self):
        self._chk(self.lib.checkpoint(self.h))

    def run(self, trace_cap=0):
        rep = Report()
        rows = np.zeros(max(trace_cap, 1), dtype=np.uint64)
        rrn = np.zeros(max(trace_cap, 1))
        X = np.empty((self.p, self.q))
        if isinstance(self.lib, OracleLib):
            code = self.lib.run(self.h, C.byref(rep), None, rrn.ctypes.data_as(_dp), None,
                                rows.ctypes.data_as(_u64p), trace_cap, _ptr(X))
        else:
            code = self.lib.run(self.h, C.byref(rep), rows.ctypes.data_as(_u64p),
                                rrn.ctypes.data_as(_dp), trace_cap, _ptr(X))
        self._chk(code)
        n = min(rep.trace_len, trace_cap)
        return rep, rows[:n].copy(), rrn[:n].copy(), X

    def greedy_threshold(self, theta):
        out = C.c_double()
        self._chk(self.lib.greedy_threshold(self.h, theta, C.byref(out)))
        return out.value

    def greedy_index_set(self, theta):
        out = np.empty(self.m, dtype=np.uint64)
        cnt = C.c_uint64()
        self._chk(self.lib.greedy_index_set(self.h, theta, out.ctypes.data_as(_u64p), C.byref(cnt)))
        return out[: cnt.value].copy()

    def max_residual_ratio(self):
        r = C.c_uint64(); v = C.c_double()
        self._chk(self.lib.max_residual_ratio(self.h, C.byref(r), C.byref(v)))
        return r.value, v.value

    def exact_metric(self):
        v = C.c_double()
        self._chk(self.lib.exact_metric(self.h, C.byref(v)))
        return v.value

    def residual_drift(self):
        v = C.c_double()
        self._chk(self.lib.residual_drift(self.h, C.byref(v)))
        return v.value

    @property
    def iteration(self):
        return self.lib.iteration(self.h)

    @property
    def alpha(self):
        return self.lib.alpha(self.h)

    @property
    def spectral_norm_b(self):
        return self.lib.spectral_norm_b(self.h)

    @property
    def residual_fro_sq(self):
        return self.lib.residual_fro_sq(self.h)

    @property
    def a_fro_sq(self):
        return self.lib.a_fro_sq(self.h)

    def current_metric(self):
        return self.lib.current_metric(self.h)

    def X(self):
        out = np.empty((self.p, self.q)); self.lib.get_X(self.h, _ptr(out)); return out

    def R(self):
        out = np.empty((self.m, self.n)); self.lib.get_R(self.h, _ptr(out)); return out

    def r_sq(self):
        out = np.empty(self.m); self.lib.get_r_sq(self.h, _ptr(out)); return out

    def a_sq(self):
        out = np.empty(self.m); self.lib.get_a_sq(self.h, _ptr(out)); return out


class PreparedSolver:
    """Oracle solver over host-precomputed caches (benchmark CPU baseline only).

    A, B, C, G = A·Aᵀ and BtB = BᵀB are borrowed (must outlive this object);
    R0 and X0 are copied.  step timing is the reference's per-iteration algorithm.
    """

    def __init__(self, lib, A, B, Cm, X0, R0, G, BtB, alpha, cfg):
        self.lib = lib
        self._keep = [np.ascontiguousarray(a, dtype=np.float64) for a in (A, B, Cm, X0, R0, G, BtB)]
        A, B, Cm, X0, R0, G, BtB = self._keep
        m, p = A.shape
        q, n = B.shape
        st = C.c_int(0)
        self.h = lib.create_prepared(_ptr(A), m, p, _ptr(B), q, n, _ptr(Cm), _ptr(X0), _ptr(R0),
                                     _ptr(G), _ptr(BtB), alpha, C.byref(cfg), C.byref(st))
        if not self.h:
            raise OracleError(st.value, "prepared create failed")
        self.cfg = cfg

    def steps(self, k):
        rows = np.empty(max(k, 1), dtype=np.uint64)
        code = self.lib.steps_c(self.h, k, rows.ctypes.data_as(_u64p))
        if code:
            raise OracleError(code, self.lib.last_error(self.h).decode())
        return rows[:k]

    def X(self):
        p, q = self._keep[0].shape[1], self._keep[1].shape[0]
        out = np.empty((p, q)); self.lib.get_X(self.h, _ptr(out)); return out

    def R(self):
        m, n = self._keep[0].shape[0], self._keep[1].shape[1]
        out = np.empty((m, n)); self.lib.get_R(self.h, _ptr(out)); return out

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.destroy(self.h)
            self.h = None


class Rng(C.Structure):
    """orc_rng — RngStream state (rng.hpp:18-123)."""

    _fields_ = [("s", C.c_uint64 * 4), ("seed", C.c_uint64), ("spare", C.c_double),
                ("has_spare", C.c_int32)]


# ---------------------------------------------------------------------------
# Reference solutions (decomp.hpp / analysis.hpp)

UNIQUE_FULL_RANK, LEAST_NORM_FULL_ROW_COL, LEAST_NORM_GENERAL = range(3)
SHAPE_ERROR, DOMAIN_ERROR = 1, 2
DECOMPOSITION_ERROR = 9


class Analysis:
    """svd / pseudoinverse / reference_solution / bk_limit / rrn through either
    the restatement (``Analysis(oracle())``) or the reference (``Analysis(ref())``)."""

    def __init__(self, lib):
        self.lib = lib
        self.is_ref = isinstance(lib, RefLib)
        S, d = C.c_size_t, C.c_double
        pre = "ref_" if self.is_ref else "orc_"
        L = lib.lib

        def f(name, args):
            fn = getattr(L, pre + name)
            fn.restype = C.c_int
            fn.argtypes = args + ([] if self.is_ref else [C.c_char_p])
            return fn

        self._svd = f("svd", [_dp, S, S, S, _dp, _dp, _dp, C.POINTER(S)])
        self._pinv = f("pseudoinverse", [_dp, S, S, d, _dp])
        self._refsol = f("reference_solution",
                         [_dp, S, S, _dp, S, S, _dp, d, _dp, C.POINTER(C.c_int), _dp])
        self._bk = f("bk_limit", [_dp, S, S, _dp, S, S, _dp, _dp, _dp])
        if self.is_ref:
            self._rrn = f("rrn", [_dp, _dp, S, S, _dp])
            L.ref_analysis_error.restype = C.c_char_p
        else:
            self._rrn = f("rrn", [_dp, _dp, S, _dp])

    def _call(self, fn, *args):
        if self.is_ref:
            code = fn(*args)
            msg = self.lib.lib.ref_analysis_error().decode() if code else ""
        else:
            buf = C.create_string_buffer(256)
            code = fn(*args, buf)
            msg = buf.value.decode()
        if code:
            raise OracleError(code, msg)

    @staticmethod
    def _c(a):
        return np.ascontiguousarray(a, dtype=np.float64)

    def svd(self, M, max_sweeps=64):
        M = self._c(M)
        rows, cols = M.shape
        r = min(rows, cols)
        U, s, V = np.empty((rows, r)), np.empty(r), np.empty((cols, r))
        rank = C.c_size_t()
        self._call(self._svd, _ptr(M), rows, cols, max_sweeps, _ptr(U), _ptr(s), _ptr(V),
                   C.byref(rank))
        return U, s, V, rank.value

    def pseudoinverse(self, M, rank_tol=-1.0):
        M = self._c(M)
        P = np.empty((M.shape[1], M.shape[0]))
        self._call(self._pinv, _ptr(M), M.shape[0], M.shape[1], rank_tol, _ptr(P))
        return P

    def reference_solution(self, A, B, Cm, rank_tol=-1.0):
        A, B, Cm = self._c(A), self._c(B), self._c(Cm)
        (m, p), (q, n) = A.shape, B.shape
        X = np.empty((p, q))
        kind, res = C.c_int(), C.c_double()
        self._call(self._refsol, _ptr(A), m, p, _ptr(B), q, n, _ptr(Cm), rank_tol, _ptr(X),
                   C.byref(kind), C.byref(res))
        return X, kind.value, res.value

    def bk_limit(self, A, B, Cm, X0):
        A, B, Cm, X0 = self._c(A), self._c(B), self._c(Cm), self._c(X0)
        (m, p), (q, n) = A.shape, B.shape
        out = np.empty((p, q))
        self._call(self._bk, _ptr(A), m, p, _ptr(B), q, n, _ptr(Cm), _ptr(X0), _ptr(out))
        return out

    def rrn(self, xk, reference):
        xk, reference = self._c(xk), self._c(reference)
        out = C.c_double()
        if self.is_ref:
            self._call(self._rrn, _ptr(xk), _ptr(reference), xk.shape[0], xk.shape[1],
                       C.byref(out))
        else:
            self._call(self._rrn, _ptr(xk), _ptr(reference), xk.size, C.byref(out))
        return out.value
