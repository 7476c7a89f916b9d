"""Error contract of the drop-in API.

Class names and base classes match the reference's errors.py:4-37 so that
`except` clauses written against `ocsc` keep catching the same failures; the
C-ABI status codes map onto them in _lib.check().
"""

# --- raised by the hot path -------------------------------------------------


class ShapeMismatchError(ValueError):
    """Extent or layout disagrees with the SignalShape (ABI status -1)."""


class DivergenceError(ArithmeticError):
    """Non-finite iterate in the code ADMM or a rejected history input (status -2)."""


class UninitializedHistoryError(RuntimeError):
    """Dictionary update asked for while the history count is zero (status -3)."""


class NumericalConsistencyError(ArithmeticError):
    """Inverse transform of a spectrum that is not Hermitian (residue guard)."""


# --- kept for API compatibility with the reference's off-path modules ------


class UndefinedVarianceError(ValueError):
    """Variance of a one-tap filter."""


class DataFileError(ValueError):
    """Root of the serialized-file errors."""


class BadMagicError(DataFileError):
    """Wrong leading tag in a serialized file."""


class ChecksumError(DataFileError):
    """Trailer checksum mismatch."""


class TruncatedFileError(DataFileError):
    """File shorter than its header promises."""
