"""Exception types with the reference's names and bases, so callers that
catch the reference exceptions keep working (eigsolve.py:21-22,
symlin.py:34-39, subqp.py:56-57, bundle.py:60-61)."""


class NumericError(RuntimeError):
    """The operator produced non-finite values."""


class ConditioningError(RuntimeError):
    """A factorization found the matrix not numerically positive definite."""


class EmptyBasisError(ValueError):
    """Orthonormalization received no usable directions."""


class StepFailureError(RuntimeError):
    """No strictly feasible step length found above the minimum."""


class FingerprintMismatch(RuntimeError):
    """A serialized state does not belong to this problem (bundle.py:60-61)."""
