"""B200-native row-action solver for A·X·B = C (arXiv 2408.05444 hot path).

Drop-in for the per-iteration path of the reference's ``axb::Solver``
(/root/reference/proj/include/axb/solver.hpp): ME-GRBK, ME-RGRBK, ME-MWRBK and the
ME-RBK / ME-BK baselines, on hand-written sm_100a CUDA behind the C-ABI in
``include/axb_b200.h``.  See DESIGN.md.
"""
from . import analysis, errors
from ._lib import LIB_PATH, device_available
from .analysis import (ReferenceCase, ReferenceSolution, SvdFactors, bk_limit, pseudoinverse,
                       reference_solution, rrn, svd)
from .errors import (CapacityError, ConfigError, ConvergenceError, CudaError, DecompositionError,
                     DivergenceError, DomainError, Error, InvariantError, ShapeError)
from .solver import (AlphaRule, Method, MethodTag, Options, SolveConfig, SolveReport, Solver,
                     StopRule, Terminated, TracePoint, kDriftGuardScale, run_many, solve,
                     trace_point_due)

__all__ = [
    "AlphaRule", "Method", "MethodTag", "Options", "SolveConfig", "SolveReport", "Solver",
    "StopRule", "Terminated", "TracePoint", "kDriftGuardScale", "solve", "trace_point_due",
    "run_many",
    "Error", "ShapeError", "DomainError", "ConfigError", "DivergenceError", "InvariantError",
    "ConvergenceError", "CapacityError", "CudaError", "DecompositionError", "errors", "LIB_PATH",
    "device_available", "analysis", "ReferenceCase", "ReferenceSolution", "SvdFactors",
    "reference_solution", "bk_limit", "rrn", "svd", "pseudoinverse",
]
