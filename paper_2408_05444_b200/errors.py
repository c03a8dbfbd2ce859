"""Exception taxonomy mirroring the reference's errors.hpp:10-72.

The C-ABI returns status codes (include/axb_b200.h); ``raise_status`` maps each
code back onto the reference exception type it stands for.
"""


class Error(RuntimeError):
    """axb::Error (errors.hpp:10-12)."""


class ShapeError(Error):
    """errors.hpp:15-17."""


class DomainError(Error):
    """errors.hpp:20-22."""


class CapacityError(Error):
    """errors.hpp:25-27 — here: device memory exhausted."""


class ConfigError(Error):
    """errors.hpp:30-32."""


class ConvergenceError(Error):
    """errors.hpp:53-57."""

    def __init__(self, msg, last_estimate=float("nan")):
        super().__init__(msg)
        self.last_estimate = last_estimate


class DivergenceError(Error):
    """errors.hpp:60-67."""

    def __init__(self, msg, iteration=0, residual_norm=float("nan")):
        super().__init__(msg)
        self.iteration = iteration
        self.residual_norm = residual_norm


class DecompositionError(Error):
    """errors.hpp:48-50 — Jacobi sweep cap, basis completion, singular LU."""


class InvariantError(Error):
    """errors.hpp:70-72."""


class CudaError(Error):
    """Device/runtime failure (no reference analogue)."""


_BY_CODE = {
    1: ShapeError,
    2: DomainError,
    3: ConfigError,
    4: DivergenceError,
    5: InvariantError,
    6: ConvergenceError,
    7: CudaError,
    8: CapacityError,
    9: DecompositionError,
}


def raise_status(code: int, msg: str, **kw):
    if code == 0:
        return
    cls = _BY_CODE.get(code, Error)
    if cls is DivergenceError:
        raise DivergenceError(msg, kw.get("iteration", 0), kw.get("residual_norm", float("nan")))
    raise cls(msg)
