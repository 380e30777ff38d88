"""numpy/scipy restatement of the reference primitives on the logm hot path.

TEST INFRASTRUCTURE (see ``oracle/__init__.py``): never imported by the product.

Each function restates the numerical behaviour of one reference routine so that,
on identical input bits, it produces identical output bits (same numpy/scipy calls
in the same order -- numpy's pairwise 1-D sums, sequential axis-0 sums, OpenBLAS
dgemm, LAPACK getrf/getrs).  The restatements additionally record decision margins
(``Margins``) that the reference does not expose; the margins are what the GPU
parity tests use to exempt near-threshold decisions.

Reference citations are relative to /root/reference/pkg/src/logmpoly/.
"""
import math

import numpy as np
import scipy.linalg

UNIT_ROUNDOFF = 2.0 ** -53            # matcore.py:19-20
SCALING_SWITCH = 1e-2                 # sqrtm.py:21
MU_MIN, MU_MAX = 1e-8, 1e8            # sqrtm.py:24


class SingularMatrixError(np.linalg.LinAlgError):
    """Exact zero pivot (exceptions.py:6)."""


class ConvergenceError(RuntimeError):
    """Iteration failed to converge (exceptions.py:10-15)."""

    def __init__(self, message, report=None):
        super().__init__(message)
        self.report = report


class Counter:
    """Work tally with the reference OpCounter's fields (matcore.py:23-48)."""

    def __init__(self):
        self.products = 0
        self.divisions = 0
        self.estimation_passes = 0


class Margins:
    """Minimum relative distance of any discrete decision from its threshold."""

    def __init__(self):
        self.min_margin = math.inf
        self.db_plateau = 0

    def cmp(self, x, thr):
        den = abs(thr)
        m = abs(x - thr) / den if den > 0 else abs(x - thr)
        if m < self.min_margin:
            self.min_margin = m

    def gap(self, a, b):
        den = max(abs(a), abs(b))
        m = abs(a - b) / den if den > 0 else 0.0
        if m < self.min_margin:
            self.min_margin = m


def _note(margins, x, thr):
    if margins is not None:
        margins.cmp(x, thr)


# ----------------------------------------------------------------------------- matcore

def as_square(A, name="matrix"):
    """Square float64 / complex128 validation (matcore.py:51-66)."""
    A = np.asarray(A)
    if A.ndim != 2 or A.shape[0] != A.shape[1] or A.shape[0] < 1:
        raise ValueError(f"{name} must be square, got shape {A.shape}")
    A = A.astype(np.complex128 if np.iscomplexobj(A) else np.float64, copy=False)
    if not np.all(np.isfinite(A.view(np.float64))):
        raise ValueError(f"{name} has non-finite entries")
    return A


def onenorm(A):
    """Max column abs-sum (matcore.py:84-87): axis-0 sum, rows accumulated in order."""
    return float(np.abs(np.asarray(A)).sum(axis=0).max())


def lu_logabsdet(A):
    """getrf + zero-pivot check + log|det| (matcore.py:94-126)."""
    A = as_square(A)
    lu, piv = scipy.linalg.lu_factor(A, check_finite=False)
    d = np.diag(lu)
    if np.any(d == 0):
        raise SingularMatrixError("matrix is exactly singular (zero pivot)")
    return (lu, piv), float(np.sum(np.log(np.abs(d))))


def lu_inverse(fac, counter=None):
    """n-column getrs against I, one division unit (matcore.py:129-148)."""
    lu, piv = fac
    n = lu.shape[0]
    if counter is not None:
        counter.divisions += 1
    return scipy.linalg.lu_solve((lu, piv), np.eye(n, dtype=lu.dtype), check_finite=False)


def balance(A, max_sweeps=100, margins=None):
    """Osborne radix-2 balancing without permutation (matcore.py:180-215).

    Returns (B, scale, sweeps) with B = T^-1 A T, T = diag(scale).
    """
    A = as_square(A)
    n = A.shape[0]
    B = A.copy()
    scale = np.ones(n)
    sweeps = 0
    for _ in range(max_sweeps):
        sweeps += 1
        moved = False
        for i in range(n):
            diag = abs(B[i, i])
            c = float(np.abs(B[:, i]).sum() - diag)
            r = float(np.abs(B[i, :]).sum() - diag)
            if c == 0.0 or r == 0.0:
                continue
            total = c + r
            f = 1.0
            while True:
                _note(margins, c, r / 2.0)
                if not c < r / 2.0:
                    break
                c *= 2.0
                r /= 2.0
                f *= 2.0
            while True:
                _note(margins, c, r * 2.0)
                if not c >= r * 2.0:
                    break
                c /= 2.0
                r *= 2.0
                f /= 2.0
            _note(margins, c + r, 0.95 * total)
            if c + r < 0.95 * total and 1e-300 < f < 1e300:
                scale[i] *= f
                B[:, i] *= f
                B[i, :] /= f
                moved = True
        if not moved:
            break
    return B, scale, sweeps


def unbalance(L, scale):
    """L -> T L T^-1 (matcore.py:175-177, 218-219)."""
    return L * (scale[:, None] / scale[None, :])


def _sign(Y):
    """matcore.py:226-231: sign(Y), and Y / |Y| (1 where Y = 0) for complex Y."""
    if np.iscomplexobj(Y):
        a = np.abs(Y)
        return np.where(a == 0, 1.0 + 0j, Y / np.where(a == 0, 1.0, a))
    return np.where(Y >= 0, 1.0, -1.0)


def est_product_norm(factors, counter=None, itmax=5, margins=None):
    """Block (t = 2) 1-norm lower bound of prod M^p (matcore.py:234-297).

    Mirrors the reference decisions exactly, including first-index argmax,
    ``argsort(-h)`` ordering, the history set and the ``h[best_j]`` row-by-column
    index quirk at matcore.py:291.
    """
    n = factors[0][0].shape[0]
    total_power = sum(p for _, p in factors)

    def forward(X):
        if counter is not None:
            counter.estimation_passes += total_power
        for M, p in factors[::-1]:
            for _ in range(p):
                X = M @ X
        return X

    def adjoint(X):
        if counter is not None:
            counter.estimation_passes += total_power
        for M, p in factors:
            Mt = M.conj().T
            for _ in range(p):
                X = Mt @ X
        return X

    t = min(2, n)
    X = np.ones((n, t)) / n
    if t > 1:
        ramp = np.array([(-1.0) ** i * (1.0 + i / max(1, n - 1)) for i in range(n)])
        X[:, 1] = ramp / np.abs(ramp).sum()
    est, best_j, seen = 0.0, 0, set()
    for sweep in range(itmax):
        Y = forward(X)
        cn = np.abs(Y).sum(axis=0)
        j = int(np.argmax(cn))
        if margins is not None and cn.shape[0] > 1:
            margins.gap(float(cn[0]), float(cn[1]))
        cand = float(cn[j])
        if margins is not None and est > 0.0:
            margins.gap(cand, est)
        if cand > est:
            est, best_j = cand, j
        elif sweep > 0:
            break
        Z = adjoint(_sign(Y))
        h = np.abs(Z).max(axis=1)
        order = np.argsort(-h)
        if margins is not None:
            hs = h[order]
            for a in range(min(len(hs) - 1, 4 * t)):
                margins.gap(float(hs[a]), float(hs[a + 1]))
        picks = [int(i) for i in order[: 4 * t] if int(i) not in seen][:t]
        if sweep > 0 and margins is not None and int(order[0]) != best_j:
            margins.gap(float(h[order[0]]), float(h[best_j]))
        if not picks or (sweep > 0 and h[order[0]] <= h[best_j]):
            break
        seen.update(picks)
        X = np.zeros((n, len(picks)))
        for c, i in enumerate(picks):
            X[i, c] = 1.0
    return est


def est_power_norm(B, p, counter=None, itmax=5, margins=None):
    """||B^p||_1 lower bound (matcore.py:300-311)."""
    if p < 1:
        raise ValueError(f"power must be a positive integer, got {p}")
    B = as_square(B)
    if not np.any(B):
        return 0.0
    return est_product_norm([(B, int(p))], counter=counter, itmax=itmax, margins=margins)


# ----------------------------------------------------------------------------- sqrtm

def sqrt_db(A, tol=None, maxiter=50, counter=None, margins=None):
    """Scaled coupled Denman-Beavers square root (sqrtm.py:27-78).

    Returns (X, iterations).  Raises SingularMatrixError / ConvergenceError /
    ValueError (non-finite iterate, via as_square inside lu_factor) like the
    reference.
    """
    A = as_square(A)
    n = A.shape[0]
    if tol is None:
        tol = 10.0 * n * UNIT_ROUNDOFF
    X = A.copy()
    Y = np.eye(n, dtype=A.dtype)  # identity_like (matcore.py:69-70): complex for complex A
    scaling = True
    for it in range(1, maxiter + 1):
        try:
            fx, lx = lu_logabsdet(X)
            fy, ly = lu_logabsdet(Y)
        except SingularMatrixError as exc:
            raise SingularMatrixError(f"singular iterate at square-root step {it}: {exc}") from exc
        mu = 1.0
        if scaling:
            mu = min(max(math.exp(-(lx + ly) / (2.0 * n)), MU_MIN), MU_MAX)
        Xi = lu_inverse(fx, counter)
        Yi = lu_inverse(fy, counter)
        Xn = 0.5 * (mu * X + Yi / mu)
        Yn = 0.5 * (mu * Y + Xi / mu)
        change = onenorm(Xn - X)
        size = onenorm(Xn)
        X, Y = Xn, Yn
        if size == 0.0:
            raise ConvergenceError("square-root iterate collapsed to zero")
        rel = change / size
        _note(margins, rel, SCALING_SWITCH)
        if rel < SCALING_SWITCH:
            scaling = False
        _note(margins, rel, tol)
        if margins is not None and tol / 10.0 <= rel <= 10.0 * tol:
            margins.db_plateau += 1
        if rel <= tol:
            return X, it
    raise ConvergenceError(f"square root did not converge in {maxiter} iterations")


# ----------------------------------------------------------------------------- schemes

def _combine(coeffs, nodes, n):
    """sum_i c_i P_i with P1 = I as a diagonal shift (schemes.py:91-101)."""
    acc = np.zeros((n, n))
    for c, P in zip(coeffs[1:], nodes):
        if c != 0.0:
            acc = acc + c * P
    if coeffs[0] != 0.0:
        acc = acc + coeffs[0] * np.eye(n)
    return acc


def eval_degopt(scheme, A, counter=None, first_product=None):
    """Degree-optimal graph polynomial (schemes.py:104-126).

    ``scheme`` = (lhs rows, rhs rows, out) as in ``paper_2401_10089_b200.constants``.
    """
    lhs, rhs, out = scheme
    A = as_square(A)
    n = A.shape[0]
    nodes = [A]
    start = 0
    if first_product is not None:
        if not (tuple(lhs[0]) == (0.0, 1.0) and tuple(rhs[0]) == (0.0, 1.0)):
            raise ValueError("first_product reuse requires a normalized scheme")
        nodes.append(first_product)
        start = 1
    for j in range(start, len(lhs)):
        left = _combine(lhs[j], nodes, n)
        right = _combine(rhs[j], nodes, n)
        if counter is not None:
            counter.products += 1
        nodes.append(left @ right)
    return _combine(out, nodes, n)
