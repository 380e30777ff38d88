"""Host-side logic of the Python layer (CPU only, no kernel launches): input validation like
``as_square`` (matcore.py:51-66), option -> C struct mapping, report decoding and exception
mapping (exceptions.py:6-18), host pipeline chunking, workspace sizing through the ABI."""
import ctypes

import numpy as np
import pytest

from paper_2401_10089_b200 import _lib, constants as C, driver
from paper_2401_10089_b200.exceptions import ConvergenceError, SingularMatrixError, SpectrumError


def test_as_batch_validation_like_as_square():
    Ab, was_numpy, squeeze = driver._as_batch(np.eye(3))
    assert Ab.shape == (1, 3, 3) and was_numpy and squeeze and Ab.dtype == np.float64
    Ab, _, squeeze = driver._as_batch(np.ones((2, 4, 4), dtype=np.float32))
    assert Ab.shape == (2, 4, 4) and not squeeze and Ab.dtype == np.float64
    for bad in (np.ones((2, 3)), np.ones((0, 0)), np.ones((2, 2, 3)), np.ones(4)):
        with pytest.raises(ValueError):
            driver._as_batch(bad)
    Ab, _, _ = driver._as_batch(np.eye(2) * (1 + 1j))     # complex128 kept (matcore.py:60-61)
    assert Ab.dtype == np.complex128


def test_c_opts_mapping():
    o, keep = driver._c_opts(driver.LogmOptions(max_k=3, maxiter=17, balance=False, db_maxiter=9, est_itmax=2))
    assert (o.max_k, o.maxiter_s, o.db_maxiter, o.est_itmax, o.balance) == (3, 17, 9, 2, 0)
    assert [o.theta[i] for i in range(C.K_MAX)] == list(C.THETA)
    th = (1e-9, 1e-5, 1e-3, 0.05, 0.2)
    o, keep = driver._c_opts(driver.LogmOptions(theta_table=th))
    assert [o.theta[i] for i in range(C.K_MAX)] == list(th) + list(C.THETA[len(th):])


def test_report_decoding_and_exception_mapping():
    rec = np.zeros(1, dtype=_lib.REPORT_DTYPE)[0]
    rec["status"], rec["s"], rec["k"], rec["products"], rec["divisions"] = 0, 3, 5, 4, 22
    rec["estimation_passes"], rec["alpha_used"], rec["min_margin"] = 90, 0.2, 1e-3
    rep = driver.LogmReport.from_record(rec)
    assert (rep.s, rep.k_selected, rep.counter.products, rep.counter.divisions) == (3, 5, 4, 22)
    assert rep.counter.equivalent_m == 4 + 4 * 22 / 3
    for status, exc in ((_lib.SINGULAR, SingularMatrixError), (_lib.DB_NOCONV, ConvergenceError),
                        (_lib.SCALING_MAXITER, ConvergenceError), (_lib.NONFINITE, ValueError),
                        (_lib.SPECTRUM, SpectrumError)):
        rec["status"] = status
        with pytest.raises(exc) as ei:
            driver._raise_for(rec, 7)
        assert "(matrix 7)" in str(ei.value)
        if exc is ConvergenceError:
            assert ei.value.report.s == 3
    assert issubclass(SingularMatrixError, np.linalg.LinAlgError)


def test_host_chunking():
    assert driver._host_chunks(100, 32) == 1
    assert driver._host_chunks(4096, 32) == 6
    assert driver._host_chunks(2000, 64) == 2
    assert driver._host_chunks(100000, 32) == 6
    assert driver._host_chunks(4096, 65) == 2       # Engine G: two stream-ordered graph chunks
    assert driver._host_chunks(40, 512) == 1        # (chunks of >= 32 matrices only)


def test_workspace_sizes_through_the_abi():
    lib = _lib.load()
    ws = ctypes.c_size_t(0)
    assert lib.lgm_workspace_bytes(32, 10, ctypes.byref(ws)) == 0 and ws.value == 10 * 8 * 32 * 32 * 8
    assert lib.lgm_workspace_bytes(64, 0, ctypes.byref(ws)) == 0 and ws.value == 0
    small, big = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.lgm_workspace_bytes(100, 16384, ctypes.byref(small)) == 0
    assert lib.lgm_workspace_bytes(100, 100000, ctypes.byref(big)) == 0
    assert big.value == small.value                  # Engine G passes reuse one workspace
    assert lib.lgm_workspace_bytes(0, 1, ctypes.byref(ws)) == _lib.ERR_ARG
