"""B200-native batched FP64 matrix logarithm (arXiv 2401.10089: inverse scaling-and-squaring
with computation-graph polynomials).

Public surface mirrors the reference ``logmpoly`` package's hot-path names
(``pkg/src/logmpoly/__init__.py:55, 60-75``): ``logm(A, opts) -> (L, LogmReport)``,
``LogmOptions``, ``LogmReport``, ``OpCounter``, ``unbalance_postprocess`` and the building
blocks ``sqrt_db``, ``est_power_norm``, ``est_product_norm``, ``balance``, ``eval_degopt``.
Everything computes on CUDA through the C ABI in include/logmpoly_b200.h; there is no CPU
fallback.  ``logm_batched`` takes (B, n, n) and shards by matrix across devices.
"""
from . import constants
from .driver import (LogmOptions, LogmReport, OpCounter, UNIT_ROUNDOFF, logm, logm_batched,
                     unbalance_postprocess)
from .exceptions import (ConvergenceError, ExtensionMissingError, SchemeFormatError, SingularMatrixError,
                         SpectrumError)
from .matio import format_matrix, parse_matrix, read_matrix, write_matrix
from .primitives import (BalanceTransform, balance, balance_batched, est_power_norm, est_product_norm,
                         eval_degopt, sqrt_db, sqrt_db_batched)
from .schemes import (GraphScheme, SchemeMeta, builtin_scheme, load_scheme, read_scheme, save_scheme,
                      write_scheme)

__version__ = "0.1.0"

__all__ = [
    "LogmOptions", "LogmReport", "OpCounter", "UNIT_ROUNDOFF", "logm", "logm_batched",
    "unbalance_postprocess", "ConvergenceError", "ExtensionMissingError", "SingularMatrixError",
    "SpectrumError", "BalanceTransform", "balance", "balance_batched", "est_power_norm",
    "est_product_norm", "eval_degopt", "sqrt_db", "sqrt_db_batched", "constants",
    "SchemeFormatError", "format_matrix", "parse_matrix", "read_matrix", "write_matrix",
    "GraphScheme", "SchemeMeta", "builtin_scheme", "load_scheme", "read_scheme", "save_scheme", "write_scheme",
]
