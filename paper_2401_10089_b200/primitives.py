"""GPU building blocks behind the C ABI, with the reference primitives' names and semantics.

Each takes a single (n, n) matrix or a (B, n, n) batch (numpy or torch), runs the
corresponding ``lgm_*_f64`` entry point and returns numpy (numpy in) or torch (torch in):

* ``sqrt_db``          <- sqrtm.py:27-78  (returns X; iterations / status via ``sqrt_db_batched``)
* ``est_power_norm``   <- matcore.py:300-311
* ``est_product_norm`` <- matcore.py:234-297 ([(M1, p1)] or [(M1, p1), (M2, 1)])
* ``balance``          <- matcore.py:180-215 (returns (B, BalanceTransform))
* ``eval_degopt``      <- schemes.py:104-126 for the shipped scheme k = 1..5
"""
import ctypes

import numpy as np

from . import _lib
from . import constants as C
from .driver import OpCounter, _as_batch, _raise_for, _torch
from .exceptions import ConvergenceError, SingularMatrixError
from .schemes import GraphScheme


class BalanceTransform:
    """Diagonal similarity T = diag(scale) (matcore.py:155-177)."""

    def __init__(self, scale):
        self.scale = np.asarray(scale, dtype=np.float64)

    @property
    def is_identity(self):
        return bool(np.all(self.scale == 1.0))

    def apply(self, A):
        return A * (self.scale[None, :] / self.scale[:, None])

    def revert(self, L):
        return L * (self.scale[:, None] / self.scale[None, :])


def _dev(A):
    torch = _torch()
    Ab, was_numpy, squeeze = _as_batch(A)
    if not torch.cuda.is_available():
        raise RuntimeError("GPU primitives need a CUDA device; there is no CPU fallback")
    if was_numpy:
        Ad = torch.from_numpy(Ab).cuda()
    else:
        Ad = Ab.to(device="cuda" if not Ab.is_cuda else Ab.device, dtype=torch.float64).contiguous()
    return Ad, was_numpy, squeeze


def _out(T, was_numpy, squeeze):
    if was_numpy:
        T = T.cpu().numpy()
    return T[0] if squeeze else T


def _stream(dev):
    return ctypes.c_void_p(_torch().cuda.current_stream(dev).cuda_stream)


def _block_ws(n, B, dev):
    """Caller-owned scratch of the building blocks (lgm_block_workspace_bytes; the library
    allocates nothing).  Returns (tensor keeping it alive, pointer, bytes)."""
    nb = ctypes.c_size_t(0)
    _lib.check(_lib.load().lgm_block_workspace_bytes(n, B, ctypes.byref(nb)), "lgm_block_workspace_bytes")
    ws = _torch().empty(max(int(nb.value), 1), dtype=_torch().uint8, device=dev)
    return ws, ws.data_ptr(), nb.value


def sqrt_db_batched(A, tol=None, maxiter=50):
    """Returns (X, iterations[int32], status[int32])."""
    torch = _torch()
    Ad, was_numpy, squeeze = _dev(A)
    B, n, _ = Ad.shape
    X = torch.empty_like(Ad)
    it = torch.zeros(B, dtype=torch.int32, device=Ad.device)
    st = torch.zeros(B, dtype=torch.int32, device=Ad.device)
    ws, wp, wb = _block_ws(n, B, Ad.device)
    _lib.check(_lib.load().lgm_sqrt_db_f64(Ad.data_ptr(), X.data_ptr(), n, B, n, float(tol or 0.0), int(maxiter),
                                           it.data_ptr(), st.data_ptr(), wp, wb, _stream(Ad.device)),
               "lgm_sqrt_db_f64")
    return _out(X, was_numpy, squeeze), it.cpu().numpy(), st.cpu().numpy()


def sqrt_db(A, tol=None, maxiter=50, counter=None):
    X, it, st = sqrt_db_batched(A, tol, maxiter)
    if counter is not None:
        counter.divisions += 2 * int(it.sum())
    bad = np.nonzero(st)[0]
    if bad.size:
        code = int(st[bad[0]])
        if code == _lib.SINGULAR:
            raise SingularMatrixError(_lib.status_string(code))
        if code == _lib.DB_NOCONV:
            raise ConvergenceError(_lib.status_string(code))
        raise ValueError(_lib.status_string(code))
    return X


def _est(M1, p1, M2, itmax, zero_shortcut):
    torch = _torch()
    Ad, was_numpy, squeeze = _dev(M1)
    B, n, _ = Ad.shape
    est = torch.zeros(B, dtype=torch.float64, device=Ad.device)
    passes = torch.zeros(B, dtype=torch.int32, device=Ad.device)
    lib = _lib.load()
    ws, wp, wb = _block_ws(n, B, Ad.device)
    if M2 is None and zero_shortcut:
        rc = lib.lgm_est_power_norm_f64(Ad.data_ptr(), n, B, n, int(p1), int(itmax), est.data_ptr(),
                                        passes.data_ptr(), wp, wb, _stream(Ad.device))
    else:
        M2d = None
        if M2 is not None:
            M2d, _, _ = _dev(M2)
        rc = lib.lgm_est_product_norm_f64(Ad.data_ptr(), int(p1), M2d.data_ptr() if M2d is not None else None, n, B,
                                          n, int(itmax), est.data_ptr(), passes.data_ptr(), wp, wb,
                                          _stream(Ad.device))
    _lib.check(rc, "lgm_est_*_norm_f64")
    e, p = est.cpu().numpy(), passes.cpu().numpy()
    return (float(e[0]), int(p[0])) if squeeze else (e, p)


def est_power_norm(B, p, counter=None, itmax=5):
    if p < 1:
        raise ValueError(f"power must be a positive integer, got {p}")
    e, passes = _est(B, p, None, itmax, True)
    if counter is not None:
        counter.estimation_passes += int(np.sum(passes))
    return e


def est_product_norm(factors, counter=None, itmax=5):
    if len(factors) == 1:
        (M1, p1), M2 = factors[0], None
    elif len(factors) == 2 and int(factors[1][1]) == 1:
        (M1, p1), (M2, _) = factors
    else:
        raise ValueError("GPU est_product_norm supports [(M1, p)] or [(M1, p), (M2, 1)]")
    e, passes = _est(M1, p1, M2, itmax, False)
    if counter is not None:
        counter.estimation_passes += int(np.sum(passes))
    return e


def balance_batched(A, max_sweeps=100):
    torch = _torch()
    Ad, was_numpy, squeeze = _dev(A)
    B, n, _ = Ad.shape
    Bo = torch.empty_like(Ad)
    sc = torch.empty((B, n), dtype=torch.float64, device=Ad.device)
    sw = torch.zeros(B, dtype=torch.int32, device=Ad.device)
    ws, wp, wb = _block_ws(n, B, Ad.device)
    _lib.check(_lib.load().lgm_balance_f64(Ad.data_ptr(), Bo.data_ptr(), sc.data_ptr(), n, B, n, int(max_sweeps),
                                           sw.data_ptr(), wp, wb, _stream(Ad.device)), "lgm_balance_f64")
    return _out(Bo, was_numpy, squeeze), sc.cpu().numpy(), sw.cpu().numpy()


def balance(A, max_sweeps=100):
    Bo, sc, _ = balance_batched(A, max_sweeps)
    if sc.shape[0] == 1 and getattr(Bo, "ndim", 3) == 2:
        return Bo, BalanceTransform(sc[0])
    return Bo, [BalanceTransform(s) for s in sc]


def eval_degopt(scheme, A, counter=None, first_product=None):
    """z(A) for a scheme (schemes.py:104-126): ``scheme`` is a GraphScheme (any coefficients,
    k <= 9 products) or an int k (the shipped scheme k)."""
    torch = _torch()
    custom = None
    if isinstance(scheme, int):
        k = scheme
    else:
        if not isinstance(scheme, GraphScheme):  # a reference-style object with lhs / rhs / out
            scheme = GraphScheme(lhs=tuple(map(tuple, scheme.lhs)), rhs=tuple(map(tuple, scheme.rhs)),
                                 out=tuple(scheme.out))
        k = scheme.mults
        if k > C.K_MAX:
            raise ValueError(f"schemes with more than {C.K_MAX} products are not supported")
        if first_product is not None and not scheme.is_normalized:
            raise ValueError("first_product reuse requires a normalized scheme")
        flat = scheme.flat()
        custom = (ctypes.c_double * len(flat))(*flat)
    Ad, was_numpy, squeeze = _dev(A)
    B, n, _ = Ad.shape
    FP = None
    if first_product is not None:
        FP, _, _ = _dev(first_product)
    Z = torch.empty_like(Ad)
    pr = torch.zeros(B, dtype=torch.int32, device=Ad.device)
    ws, wp, wb = _block_ws(n, B, Ad.device)
    lib = _lib.load()
    fp = FP.data_ptr() if FP is not None else None
    if custom is None:
        rc = lib.lgm_eval_degopt_f64(Ad.data_ptr(), fp, Z.data_ptr(), n, B, n, k, pr.data_ptr(), wp, wb,
                                     _stream(Ad.device))
    else:
        rc = lib.lgm_eval_degopt_scheme_f64(Ad.data_ptr(), fp, Z.data_ptr(), n, B, n, k, custom, pr.data_ptr(), wp,
                                            wb, _stream(Ad.device))
    _lib.check(rc, "lgm_eval_degopt")
    if counter is not None:
        counter.products += int(pr.cpu().numpy().sum())
    return _out(Z, was_numpy, squeeze)


__all__ = ["BalanceTransform", "OpCounter", "balance", "balance_batched", "est_power_norm",
           "est_product_norm", "eval_degopt", "sqrt_db", "sqrt_db_batched", "_raise_for"]
