"""Error types of the B200 rapid-Kriging package.

Class names match the reference package (rapidkrig errors.py:4-17) so callers'
``except`` clauses keep working; the C ABI's rk_status codes map onto them in
``_native.check``:  RK_DOMAIN -> DomainError, RK_NUMERIC -> NumericError,
RK_INTERNAL -> InternalError, RK_CUDA -> RapidKrigError.
"""


class RapidKrigError(Exception):
    pass


class DomainError(RapidKrigError):
    """Bad arguments: shapes, parameter ranges, locations outside the grid."""


class NumericError(RapidKrigError):
    """Factorisation, series convergence or embedding positivity failed."""


class InternalError(RapidKrigError):
    """Broken internal invariant (e.g. a stencil leaving the padded grid)."""
