"""ctypes binding of the C ABI in include/logmpoly_b200.h (the library is built in-tree by
``make`` / ``__graft_entry__.build()`` into ``_build/liblogmpoly_b200.so``).

The library is loaded lazily on first use so that the package imports on CPU-only hosts;
any attempt to compute without it raises ``ExtensionMissingError`` -- there is no CPU
fallback anywhere in the product.
"""
import ctypes
import os

import numpy as np

from .exceptions import ExtensionMissingError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "liblogmpoly_b200.so")

# status codes (lgm_report.status)
OK, SINGULAR, DB_NOCONV, SCALING_MAXITER, NONFINITE, SPECTRUM = 0, 1, 2, 3, 4, 5
ERR_ARG, ERR_CUDA, ERR_UNSUPPORTED, ERR_WORKSPACE = -1, -2, -3, -4

# every symbol include/logmpoly_b200.h declares
EXPORTS = ("lgm_default_opts", "lgm_workspace_bytes", "lgm_block_workspace_bytes", "lgm_max_fused_n", "lgm_logm_f64",
           "lgm_sqrt_db_f64", "lgm_est_power_norm_f64", "lgm_est_product_norm_f64",
           "lgm_balance_f64", "lgm_eval_degopt_f64", "lgm_expm_ref_f64", "lgm_spectrum_check_f64", "lgm_status_string", "lgm_launch_count",
           "lgm_debug_ws_guard", "lgm_eval_degopt_scheme_f64")


class Opts(ctypes.Structure):
    _fields_ = [("max_k", ctypes.c_int32), ("maxiter_s", ctypes.c_int32),
                ("db_maxiter", ctypes.c_int32), ("est_itmax", ctypes.c_int32),
                ("balance", ctypes.c_int32), ("embedded_complex", ctypes.c_int32),
                ("db_tol", ctypes.c_double), ("theta", ctypes.POINTER(ctypes.c_double))]


REPORT_DTYPE = np.dtype([("status", "<i4"), ("s", "<i4"), ("k", "<i4"), ("db_iters", "<i4"),
                         ("products", "<i4"), ("divisions", "<i4"), ("estimation_passes", "<i4"),
                         ("norm_estimations", "<i4"), ("balanced", "<i4"), ("balance_sweeps", "<i4"),
                         ("db_plateau", "<i4"), ("inv_skipped", "<i4"), ("alpha_used", "<f8"), ("min_margin", "<f8")])
assert REPORT_DTYPE.itemsize == 64

_lib = None

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32


def load(path=LIB_PATH):
    """Load (once) and return the CDLL with argtypes set."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ExtensionMissingError(
            f"{path} not built: run `make` (or __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(path)
    lib.lgm_default_opts.argtypes = [ctypes.POINTER(Opts)]
    lib.lgm_default_opts.restype = None
    lib.lgm_workspace_bytes.argtypes = [_I64, _I64, ctypes.POINTER(ctypes.c_size_t)]
    lib.lgm_max_fused_n.argtypes = []
    lib.lgm_logm_f64.argtypes = [_P, _P, _I64, _I64, _I64, ctypes.POINTER(Opts), _P, _P,
                                 ctypes.c_size_t, _P]
    lib.lgm_block_workspace_bytes.argtypes = [_I64, _I64, ctypes.POINTER(ctypes.c_size_t)]
    _W = ctypes.c_size_t
    lib.lgm_sqrt_db_f64.argtypes = [_P, _P, _I64, _I64, _I64, ctypes.c_double, _I32, _P, _P, _P, _W, _P]
    lib.lgm_est_power_norm_f64.argtypes = [_P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P, _W, _P]
    lib.lgm_est_product_norm_f64.argtypes = [_P, _I32, _P, _I64, _I64, _I64, _I32, _P, _P, _P, _W, _P]
    lib.lgm_balance_f64.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I32, _P, _P, _W, _P]
    lib.lgm_eval_degopt_f64.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I32, _P, _P, _W, _P]
    lib.lgm_eval_degopt_scheme_f64.argtypes = [_P, _P, _P, _I64, _I64, _I64, _I32, _P, _P, _P, _W, _P]
    lib.lgm_expm_ref_f64.argtypes = [_P, _P, _I64, _I64, _I64, _P, _W, _P]
    lib.lgm_spectrum_check_f64.argtypes = [_P, _P, _I64, _I64, _I64, _P, _W, _P]
    lib.lgm_status_string.argtypes = [ctypes.c_int]
    lib.lgm_status_string.restype = ctypes.c_char_p
    lib.lgm_debug_ws_guard.argtypes = [_I64, _I64, _I32, _P, _I32, _P, _P]
    lib.lgm_launch_count.argtypes = []
    lib.lgm_launch_count.restype = ctypes.c_longlong
    for name in EXPORTS:
        if name not in ("lgm_default_opts", "lgm_status_string", "lgm_launch_count"):
            getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def launch_count():
    return int(load().lgm_launch_count())


def status_string(code):
    return load().lgm_status_string(int(code)).decode()


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed: {status_string(rc)} ({rc})")
