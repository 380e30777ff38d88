"""Benchmark / accuracy harness around the GPU logm.

The reference's bench/CLI layer is specified but missing (``logmpoly/__init__.py:56``); this is
the caller side of the hot path, restated from the SPEC's ``cli`` module:

* ``relative_error`` -- Er = ||L_hat - L_ref||_2 / ||L_ref||_2 (PAPER section 7); the 2-norm is
  an exact SVD for n <= 64 and 50 steps of power iteration on M^T M (tol 1e-10) above
  (SPEC.md:541).  ``relative_error_batched`` does the same for (B, n, n) tensors on the GPU
  (torch plumbing, not the product path).
* ``performance_profile`` -- Dolan-More curves p(alpha), alpha = 1.0, 1.1, ..., 5.0, on
  errors floored at the unit roundoff, Er' = max(Er, u) (ledger decision).
* ``gen_test_matrices`` -- the SPEC's four deterministic families:
  (a) I + A with ||A||_2 = 0.5, (b) known log V diag(e^lambda) V^-1 (shipped with its log),
  (c) non-normal I + scaled upper bidiagonal, (d) SPD Q^T D Q.
* ``BenchRecord`` / ``run_bench`` / CSV round trip (17 significant digits).

Everything that computes a logarithm goes through ``logm_batched`` (CUDA, no CPU fallback).
"""
import csv
import io
import time
from dataclasses import asdict, dataclass, fields

import numpy as np

UNIT_ROUNDOFF = 2.0 ** -53
PROFILE_ALPHAS = tuple(round(1.0 + 0.1 * i, 1) for i in range(41))


# ----------------------------------------------------------------------------- 2-norms

def _power_norm2(M, steps=50, tol=1e-10):
    """sigma_max(M) by power iteration on M^T M from a fixed start vector."""
    n = M.shape[1]
    x = np.full(n, 1.0 / np.sqrt(n))
    sig = 0.0
    for _ in range(steps):
        y = M.T @ (M @ x)
        ny = np.linalg.norm(y)
        if ny == 0.0:
            return 0.0
        x = y / ny
        new = np.sqrt(ny)
        if sig > 0.0 and abs(new - sig) <= tol * new:
            sig = new
            break
        sig = new
    return float(np.linalg.norm(M @ x)) if sig > 0.0 else 0.0


def norm2(M):
    """Spectral norm with the SPEC's method choice (SVD for n <= 64, power iteration above)."""
    M = np.asarray(M, dtype=np.float64)
    if M.shape[-1] <= 64:
        return float(np.linalg.norm(M, 2))
    return _power_norm2(M)


def relative_error(L_hat, L_ref):
    """Er(A) = ||L_hat - L_ref||_2 / ||L_ref||_2; L_ref = 0 is undefined."""
    L_hat = np.asarray(L_hat, dtype=np.float64)
    L_ref = np.asarray(L_ref, dtype=np.float64)
    den = norm2(L_ref)
    if den == 0.0:
        raise ValueError("relative error undefined for a zero reference logarithm")
    return norm2(L_hat - L_ref) / den


def relative_error_batched(L_hat, L_ref, steps=50, tol=1e-10):
    """Er per matrix for (B, n, n) torch tensors on their device (same method choice)."""
    import torch
    D = (L_hat - L_ref).to(torch.float64)
    R = L_ref.to(torch.float64)
    if D.shape[-1] <= 64:
        num = torch.linalg.matrix_norm(D, ord=2)
        den = torch.linalg.matrix_norm(R, ord=2)
    else:
        def pw(M):
            n = M.shape[-1]
            x = torch.full((M.shape[0], n, 1), 1.0 / n ** 0.5, dtype=M.dtype, device=M.device)
            sig = torch.zeros(M.shape[0], dtype=M.dtype, device=M.device)
            Mt = M.transpose(-1, -2)
            for _ in range(steps):
                y = Mt @ (M @ x)
                ny = torch.linalg.vector_norm(y, dim=(-2, -1))
                x = y / torch.where(ny > 0, ny, torch.ones_like(ny))[:, None, None]
                new = ny.sqrt()
                done = (sig > 0) & ((new - sig).abs() <= tol * new)
                sig = new
                if bool(done.all()):
                    break
            return torch.linalg.vector_norm(M @ x, dim=(-2, -1))
        num, den = pw(D), pw(R)
    if bool((den == 0).any()):
        raise ValueError("relative error undefined for a zero reference logarithm")
    return (num / den).cpu().numpy()


# ----------------------------------------------------------------------------- profiles

def performance_profile(errors, alphas=PROFILE_ALPHAS, floor=UNIT_ROUNDOFF):
    """Dolan-More performance profile of relative errors.

    ``errors``: {matrix_id: {method: Er}}; every matrix must carry every method.  Returns
    {method: [(alpha, p), ...]} with p = fraction of matrices whose floored error
    Er' = max(Er, floor) is <= alpha * min over methods of Er'.
    """
    if not errors:
        raise ValueError("no records")
    methods = sorted({m for rec in errors.values() for m in rec})
    for mid, rec in errors.items():
        missing = [m for m in methods if m not in rec]
        if missing:
            raise ValueError(f"incomplete record grid: matrix {mid!r} lacks {missing}")
    E = np.array([[max(float(errors[mid][m]), floor) for m in methods] for mid in errors])
    ratio = E / E.min(axis=1, keepdims=True)
    return {m: [(a, float(np.mean(ratio[:, j] <= a * (1.0 + 1e-12)))) for a in alphas]
            for j, m in enumerate(methods)}


# ----------------------------------------------------------------------------- matrices

def _orth(rng, n):
    Q, R = np.linalg.qr(rng.standard_normal((n, n)))
    return Q * np.sign(np.diag(R))[None, :]


def gen_test_matrices(family, seed, n, count=1, kappa=10.0, superdiag=None):
    """Deterministic synthetic families.  Returns (A[count, n, n], L_ref or
    None): only family "b" (known log) ships its reference logarithm.

    a: I + A, A Gaussian scaled to ||A||_2 = 0.5 (the paper's introduction example);
    b: V diag(e^lambda) V^-1, lambda in [-1, 1], cond_2(V) = kappa, L_ref = V diag(lambda) V^-1;
    c: I + s * (upper bidiagonal with unit superdiagonal), s = superdiag or U(0.5, 5);
    d: SPD Q^T D Q with D log-uniform in [1e-2, 1e2].
    """
    rng = np.random.default_rng(seed)
    A = np.empty((count, n, n))
    L = np.empty((count, n, n)) if family == "b" else None
    for q in range(count):
        if family == "a":
            G = rng.standard_normal((n, n))
            A[q] = np.eye(n) + 0.5 * G / np.linalg.norm(G, 2)
        elif family == "b":
            U, W = _orth(rng, n), _orth(rng, n)
            V = (U * np.logspace(0.0, np.log10(kappa), n)[None, :]) @ W.T
            lam = rng.uniform(-1.0, 1.0, n)
            Vi = np.linalg.inv(V)
            A[q] = (V * np.exp(lam)[None, :]) @ Vi
            L[q] = (V * lam[None, :]) @ Vi
        elif family == "c":
            s = superdiag if superdiag is not None else rng.uniform(0.5, 5.0)
            A[q] = np.eye(n) + s * np.eye(n, k=1)
        elif family == "d":
            Q = _orth(rng, n)
            d = 10.0 ** rng.uniform(-2.0, 2.0, n)
            M = (Q.T * d[None, :]) @ Q
            A[q] = 0.5 * (M + M.T)
        else:
            raise ValueError(f"unknown family {family!r} (a, b, c, d)")
    return A, L


# ----------------------------------------------------------------------------- records

@dataclass
class BenchRecord:
    """One (matrix, method) result."""

    matrix_id: str
    n: int
    method: str
    er: float
    products: int
    divisions: int
    equivalent_m: float
    wall_s: float
    status: int = 0
    s: int = 0
    k: int = 0


def records_to_csv(records):
    """CSV with a header row and 17 significant digits for floats."""
    out = io.StringIO()
    names = [f.name for f in fields(BenchRecord)]
    w = csv.writer(out, lineterminator="\n")
    w.writerow(names)
    for r in records:
        d = asdict(r)
        w.writerow([f"{d[k]:.17g}" if isinstance(d[k], float) else d[k] for k in names])
    return out.getvalue()


def records_from_csv(text):
    rows = list(csv.reader(io.StringIO(text)))
    if not rows:
        raise ValueError("empty CSV")
    names = rows[0]
    types = {f.name: f.type for f in fields(BenchRecord)}
    conv = {"int": int, "float": float, "str": str, int: int, float: float, str: str}
    out = []
    for row in rows[1:]:
        out.append(BenchRecord(**{k: conv[types[k]](v) for k, v in zip(names, row)}))
    return out


def run_bench(A, L_ref=None, method="logm_graph_b200", ids=None, opts=None):
    """Run the GPU logm over a (B, n, n) set and return one BenchRecord per matrix.

    Er is measured against ``L_ref`` when given (family b), else NaN.  ``wall_s`` is the
    batch wall time divided evenly (matrices run concurrently on the device).
    """
    import torch
    from . import driver
    opts = opts or driver.LogmOptions(raise_on_error=False)
    A = np.ascontiguousarray(A, dtype=np.float64)
    B, n, _ = A.shape
    ids = ids or [f"m{q:04d}" for q in range(B)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    L, reps = driver.logm_batched(A, opts)
    wall = (time.perf_counter() - t0) / max(B, 1)
    er = np.full(B, np.nan)
    ok = reps["status"] == 0
    if L_ref is not None and ok.any():
        er[ok] = relative_error_batched(torch.from_numpy(np.asarray(L)[ok]).cuda(),
                                        torch.from_numpy(np.asarray(L_ref)[ok]).cuda())
    recs = []
    for q in range(B):
        r = reps[q]
        recs.append(BenchRecord(matrix_id=ids[q], n=n, method=method, er=float(er[q]),
                                products=int(r["products"]), divisions=int(r["divisions"]),
                                equivalent_m=float(r["products"] + 4.0 * r["divisions"] / 3.0),
                                wall_s=wall, status=int(r["status"]), s=int(r["s"]), k=int(r["k"])))
    return recs, L
