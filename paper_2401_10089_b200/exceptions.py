"""Exception types of the hot path, same names/bases as the reference's
``logmpoly/exceptions.py:6-18`` so that callers' ``except`` clauses keep working."""
import numpy as np


class SingularMatrixError(np.linalg.LinAlgError):
    """Exact zero pivot in a square-root step (matcore.py:124-125, sqrtm.py:51-56)."""


class ConvergenceError(RuntimeError):
    """DB iteration or scaling loop hit its cap (sqrtm.py:76-78); carries the report."""

    def __init__(self, message, report=None):
        super().__init__(message)
        self.report = report


class SpectrumError(ValueError):
    """Eigenvalues on the closed negative real axis (exceptions.py:18)."""


class ExtensionMissingError(RuntimeError):
    """The CUDA shared library is not built / not loadable.  There is no CPU fallback."""


class SchemeFormatError(ValueError):
    """A matrix (or coefficient) text file could not be parsed (exceptions.py:22)."""
