"""Reference solutions on the B200 — analysis.hpp / decomp.hpp mirror.

The reference produces the X* that ``StopRule.solution_rrn`` and the benchmark
harness compare against with host code: ``reference_solution`` (analysis.hpp:48-91),
``bk_limit`` (:95-104), ``rrn`` (:107-111), on top of ``svd`` (decomp.hpp:113-157,
one-sided cyclic Jacobi) and ``pseudoinverse`` (:161-177).  Here the same API runs
on the device (csrc/axb_analysis.cu): round-robin parallel Jacobi, one CTA per
column pair, and DMMA GEMMs for A⁺, (A⁺·C)·B⁺ and the consistency guard.

Same names, argument meanings and exceptions as the reference: ShapeError for
an empty operand, DecompositionError when Jacobi hits its sweep cap, DomainError
for an inconsistent system or a zero rrn reference.  Operands are numpy arrays
(dense) or scipy CSR matrices (expanded like ``to_dense``).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .errors import raise_status

kConsistencyGuardScale = 1e-8  # analysis.hpp:16


class ReferenceCase(enum.IntEnum):  # analysis.hpp:18
    UniqueFullRank = 0
    LeastNormFullRowCol = 1
    LeastNormGeneral = 2


def reference_case_label(c: ReferenceCase) -> str:  # analysis.hpp:20-28
    return {ReferenceCase.UniqueFullRank: "unique_full_rank",
            ReferenceCase.LeastNormFullRowCol: "least_norm_full_row_col",
            ReferenceCase.LeastNormGeneral: "least_norm_general"}.get(c, "?")


@dataclass
class ReferenceSolution:  # analysis.hpp:30-34
    X_star: np.ndarray
    kind: ReferenceCase
    residual_check: float


@dataclass
class SvdFactors:  # decomp.hpp:15-27
    U: Optional[np.ndarray]
    singular_values: np.ndarray
    V: Optional[np.ndarray]
    numeric_rank: int

    def sigma_max(self) -> float:
        return float(self.singular_values[0]) if self.singular_values.size else 0.0

    def sigma_min_positive(self) -> float:
        r = self.numeric_rank
        return 0.0 if r == 0 else float(self.singular_values[r - 1])


def default_rank_tol(rows: int, cols: int, sigma_max: float) -> float:  # decomp.hpp:30-33
    return 8.0 * float(max(rows, cols)) * sigma_max * 2.0 ** -52


def _dense(M):
    if hasattr(M, "tocsr"):
        M = M.toarray()
    return np.ascontiguousarray(M, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(_lib._dp)


def _check(st):
    if st:
        raise_status(st, _lib.load().axb_last_create_error().decode())


def _desc(M, keep):
    """axb_matrix for a dense array or a scipy CSR matrix."""
    d = _lib.AxbMatrix()
    d.rows, d.cols = M.shape
    if hasattr(M, "tocsr"):
        M = M.tocsr()
        M.sort_indices()
        rp = np.ascontiguousarray(M.indptr, dtype=np.uint64)
        ci = np.ascontiguousarray(M.indices, dtype=np.uint64)
        vv = np.ascontiguousarray(M.data, dtype=np.float64)
        keep.extend([rp, ci, vv])
        d.kind, d.nnz = 1, vv.size
        d.row_ptr, d.col_idx, d.values = rp.ctypes.data, ci.ctypes.data, vv.ctypes.data
    else:
        a = _dense(M)
        keep.append(a)
        d.kind = 0
        d.dense = a.ctypes.data
    return d


def svd(M, max_sweeps: int = 64, *, compute_uv: bool = True, device: int = 0) -> SvdFactors:
    """decomp.hpp:113-157 on the device.  U is rows×r, V cols×r, r = min(rows, cols)."""
    lib = _lib.load()
    M = _dense(M)
    rows, cols = M.shape
    r = min(rows, cols)
    s = np.empty(r)
    U = np.empty((rows, r)) if compute_uv else None
    V = np.empty((cols, r)) if compute_uv else None
    rank = C.c_uint64()
    _check(lib.axb_svd(_p(M), rows, cols, max_sweeps, device, _p(U), _p(s), _p(V),
                       C.byref(rank)))
    return SvdFactors(U, s, V, int(rank.value))


def pseudoinverse(M, rank_tol: float = -1.0, *, device: int = 0) -> np.ndarray:
    """decomp.hpp:161-177: the cols×rows Moore–Penrose pseudoinverse."""
    lib = _lib.load()
    M = _dense(M)
    rows, cols = M.shape
    P = np.empty((cols, rows))
    _check(lib.axb_pseudoinverse(_p(M), rows, cols, float(rank_tol), device, _p(P)))
    return P


def reference_solution(A, B, C_, rank_tol: float = -1.0, *, device: int = 0) -> ReferenceSolution:
    """analysis.hpp:48-91: X* with its ReferenceCase and ‖A·X*·B − C‖_F."""
    lib = _lib.load()
    keep = []
    dA, dB = _desc(A, keep), _desc(B, keep)
    Cm = _dense(C_)
    p, q = A.shape[1], B.shape[0]
    X = np.empty((p, q))
    kind, res = C.c_int32(), C.c_double()
    _check(lib.axb_reference_solution(C.byref(dA), C.byref(dB), _p(Cm), float(rank_tol), device,
                                      _p(X), C.byref(kind), C.byref(res)))
    return ReferenceSolution(X, ReferenceCase(kind.value), res.value)


def bk_limit(A, B, C_, X0, *, device: int = 0) -> np.ndarray:
    """analysis.hpp:95-104: the point ME-BK converges to from X0."""
    lib = _lib.load()
    keep = []
    dA, dB = _desc(A, keep), _desc(B, keep)
    Cm, X0 = _dense(C_), _dense(X0)
    out = np.empty((A.shape[1], B.shape[0]))
    _check(lib.axb_bk_limit(C.byref(dA), C.byref(dB), _p(Cm), _p(X0), device, _p(out)))
    return out


def rrn(xk, reference, *, device: int = 0) -> float:
    """analysis.hpp:107-111: ‖Xk − ref‖²_F / ‖ref‖²_F."""
    lib = _lib.load()
    a, b = _dense(xk), _dense(reference)
    if a.shape != b.shape:
        raise_status(1, "sub: shape mismatch")
    out = C.c_double()
    _check(lib.axb_rrn(_p(a), _p(b), a.size, device, C.byref(out)))
    return out.value


def last_stats():
    """(Jacobi sweeps of A, of B, device ms) of this thread's last analysis call."""
    sw = (C.c_uint64 * 2)()
    ms = C.c_double()
    _lib.load().axb_analysis_stats(C.cast(sw, _lib._u64p), C.byref(ms))
    return int(sw[0]), int(sw[1]), ms.value
