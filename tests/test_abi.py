"""CPU-side checks of the C-ABI boundary: the library builds, loads and exports every symbol
include/logmpoly_b200.h declares; host-only entry points behave (no compute without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2401_10089_b200 import _lib
from paper_2401_10089_b200 import constants as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_symbols():
    text = open(os.path.join(ROOT, "include", "logmpoly_b200.h")).read()
    return sorted(set(re.findall(r"\b(lgm_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = _header_symbols()
    assert set(syms) == set(_lib.EXPORTS)
    for s in syms:
        assert hasattr(lib, s), s


def test_default_opts_and_workspace():
    lib = _lib.load()
    o = _lib.Opts()
    lib.lgm_default_opts(ctypes.byref(o))
    assert (o.max_k, o.maxiter_s, o.db_maxiter, o.est_itmax, o.balance) == (C.K_DEFAULT, 40, 50, 5, 1)
    assert o.db_tol == 0.0 and not o.theta
    ws = ctypes.c_size_t(123)
    # fused engine: 8 n^2 doubles per matrix (polynomial nodes P4..P10 and A_I2)
    assert lib.lgm_workspace_bytes(32, 4096, ctypes.byref(ws)) == 0 and ws.value == 4096 * 8 * 32 * 32 * 8
    assert lib.lgm_workspace_bytes(512, 2, ctypes.byref(ws)) == 0 and ws.value >= 2 * 12 * 512 * 512 * 8
    assert lib.lgm_launch_count() >= 0
    assert lib.lgm_block_workspace_bytes(32, 8, ctypes.byref(ws)) == 0 and ws.value > 0
    assert lib.lgm_block_workspace_bytes(100, 8, ctypes.byref(ws)) == 0 and ws.value >= 8 * 8 * 100 * 100 * 8
    assert lib.lgm_workspace_bytes(0, 1, ctypes.byref(ws)) == _lib.ERR_ARG
    assert lib.lgm_max_fused_n() == 64


def test_status_strings_and_argument_errors():
    assert "singular" in _lib.status_string(_lib.SINGULAR)
    assert "converge" in _lib.status_string(_lib.DB_NOCONV)
    assert "non-finite" in _lib.status_string(_lib.NONFINITE)
    lib = _lib.load()
    # argument validation happens before any CUDA call
    assert lib.lgm_logm_f64(None, None, 4, 1, 4, None, None, None, 0, None) == _lib.ERR_ARG
    assert lib.lgm_logm_f64(1, 2, 4, 1, 3, None, 3, None, 0, None) == _lib.ERR_ARG  # ld < n


def test_report_layout_matches_header():
    assert _lib.REPORT_DTYPE.itemsize == 64
    assert ctypes.sizeof(_lib.Opts) == 40


def test_no_cpu_fallback():
    import torch
    from paper_2401_10089_b200 import logm
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        logm(np.eye(3))


def test_constants_match_c_header():
    from paper_2401_10089_b200 import constants as C
    text = open(os.path.join(ROOT, "paper_2401_10089_b200", "csrc", "lgm_constants.h")).read()
    th = re.search(r"LGM_THETA_DEFAULT\[LGM_K_MAX\] = \{([^}]*)\}", text).group(1)
    assert tuple(float(x) for x in th.split(",")) == C.THETA
