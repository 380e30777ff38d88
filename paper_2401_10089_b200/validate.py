"""On-device validation helpers: batched reference exponential and the
spectrum pre-check.

* ``expm_ref_batched(A)`` runs the reference's test-oracle exponential
  (``logmpoly/matcore.py:318-336``) as the library's own kernels (``lgm_expm_ref_f64``:
  device-side scaling exponent from the 1-norm, 20 Horner DMMA GEMMs T = I + X T / j with the
  division and identity fused into the epilogue, squarings in a device-driven CUDA-graph loop,
  per matrix s) -- no cuBLAS, no host round trip.
* ``spectrum_violations(A, cap=512)`` is the principal-logarithm precondition check of
  ``eig_small`` (``matcore.py:343-355``): True where a matrix has an
  eigenvalue on the closed negative real axis.  Matrices above ``cap`` are not checked (the
  SPEC's cap: there violations surface as DB non-convergence).
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


def spectrum_violations(A, cap=512):
    """Boolean mask (numpy, per matrix): an eigenvalue lies on the closed negative real axis
    (real eigenvalue <= 0).  Matrices with n > cap are reported False (unchecked)."""
    torch = _torch()
    if not isinstance(A, torch.Tensor):
        A = torch.from_numpy(np.ascontiguousarray(A, dtype=np.float64))
    if A.dim() == 2:
        A = A.unsqueeze(0)
    if A.shape[-1] > cap:
        return np.zeros(A.shape[0], dtype=bool)
    lam = torch.linalg.eigvals(A.to(torch.float64))
    bad = (lam.imag == 0) & (lam.real <= 0)
    return bad.any(dim=-1).cpu().numpy()
