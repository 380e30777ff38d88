"""On-device validation helpers: batched reference exponential and the
spectrum pre-check.  Both are torch plumbing on the GPU (cuBLAS / cuSOLVER), not the product
path; they exist to validate it.

* ``expm_ref_batched(A)`` restates the reference's test-oracle exponential
  (``logmpoly/matcore.py:316-334``): scale by 2^-s so that ||A||_1 <= 1/2, degree-20 Taylor
  polynomial in Horner form T = I + X T / j (j = 20..1), then s squarings -- per matrix s,
  batched.
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
    """exp of each (n, n) block of a (B, n, n) float64 CUDA tensor (matcore.py:316-334)."""
    torch = _torch()
    A = A.to(torch.float64)
    B, n, _ = A.shape
    nrm = A.abs().sum(dim=-2).amax(dim=-1).cpu().numpy()          # ||A||_1 per matrix
    s = np.array([0 if v <= 0.5 else max(0, int(math.ceil(math.log2(v / 0.5)))) for v in nrm])
    scale = torch.from_numpy(np.ldexp(1.0, -s)).to(A.device)
    X = A * scale[:, None, None]
    eye = torch.eye(n, dtype=A.dtype, device=A.device).expand(B, n, n)
    T = eye.clone()
    for j in range(20, 0, -1):
        T = eye + (X @ T) / j
    for i in range(int(s.max()) if B else 0):
        sq = torch.from_numpy(s > i).to(A.device)
        T = torch.where(sq[:, None, None], T @ T, T)
    return T


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
