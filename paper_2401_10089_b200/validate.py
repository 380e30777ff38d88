"""On-device validation helpers: batched reference exponential and the
spectrum pre-check.

* ``expm_ref_batched(A)`` runs the reference's test-oracle exponential
  (``logmpoly/matcore.py:318-336``) as the library's own kernels (``lgm_expm_ref_f64``:
  device-side scaling exponent from the 1-norm, 20 Horner DMMA GEMMs T = I + X T / j with the
  division and identity fused into the epilogue, squarings in a device-driven CUDA-graph loop,
  per matrix s) -- no cuBLAS, no host round trip.
* ``spectrum_violations(A, cap=512)`` is the principal-logarithm precondition check of
  ``eig_small`` (``matcore.py:343-355``): True where a matrix has an
  eigenvalue on the closed negative real axis, decided by the library's own kernel
  (``lgm_spectrum_check_f64``: Householder Hessenberg reduction + Francis double-shift QR, one
  CTA per matrix).  Matrices above ``cap`` are not checked (the SPEC's cap: there violations
  surface as DB non-convergence).
"""
import math

import numpy as np


def _torch():
    import torch
    return torch


def expm_ref_batched(A):
    """exp of each (n, n) block of a (B, n, n) float64 CUDA tensor (matcore.py:318-336), on the
    library's kernels (lgm_expm_ref_f64)."""
    import ctypes
    from . import _lib
    torch = _torch()
    A = A.to(torch.float64).contiguous()
    if A.dim() == 2:
        A = A.unsqueeze(0)
    B, n, _ = A.shape
    E = torch.empty_like(A)
    lib = _lib.load()
    nb = ctypes.c_size_t(0)
    _lib.check(lib.lgm_block_workspace_bytes(n, B, ctypes.byref(nb)), "lgm_block_workspace_bytes")
    stream = torch.cuda.current_stream(A.device)
    with torch.cuda.stream(stream):
        ws = torch.empty(max(int(nb.value), 1), dtype=torch.uint8, device=A.device)
    _lib.check(lib.lgm_expm_ref_f64(A.data_ptr(), E.data_ptr(), n, B, n, ws.data_ptr(), nb.value,
                                    ctypes.c_void_p(stream.cuda_stream)), "lgm_expm_ref_f64")
    return E


def spectrum_check(A):
    """Per-matrix flags of lgm_spectrum_check_f64 (the library's Hessenberg + Francis QR):
    1 = an eigenvalue on the closed negative real axis, 0 = none, 2 = QR did not converge."""
    import ctypes
    from . import _lib
    torch = _torch()
    if not isinstance(A, torch.Tensor):
        A = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64))
    if A.dim() == 2:
        A = A.unsqueeze(0)
    dev = A.device if A.is_cuda else torch.device("cuda", torch.cuda.current_device())
    A = A.to(device=dev, dtype=torch.float64).contiguous()
    B, n, _ = A.shape
    flags = torch.zeros(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    nb = B * n * n * 8
    with torch.cuda.stream(stream):
        ws = torch.empty(max(nb, 1), dtype=torch.uint8, device=dev)
    _lib.check(_lib.load().lgm_spectrum_check_f64(A.data_ptr(), flags.data_ptr(), n, B, n, ws.data_ptr(), nb,
                                                  ctypes.c_void_p(stream.cuda_stream)), "lgm_spectrum_check_f64")
    return flags.cpu().numpy()


def spectrum_violations(A, cap=512):
    """Boolean mask (numpy, per matrix): an eigenvalue lies on the closed negative real axis
    (real eigenvalue <= 0), decided on the device (spectrum_check).  Matrices with n > cap are
    reported False (unchecked, as eig_small's cap); a QR non-convergence raises
    ConvergenceError like eig_small (matcore.py:353-355)."""
    from .exceptions import ConvergenceError
    torch = _torch()
    n = A.shape[-1]
    if n > cap:
        B = A.shape[0] if len(A.shape) == 3 else 1
        return np.zeros(B, dtype=bool)
    f = spectrum_check(A)
    if (f == 2).any():
        raise ConvergenceError("eigenvalue iteration failed (spectrum pre-check)", None)
    return f == 1
