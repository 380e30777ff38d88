"""Restated Algorithm 1 (inverse scaling-and-squaring logm) -- TEST INFRASTRUCTURE ONLY.

The reference's driver module (``logmpoly/driver.py``) is imported at
``logmpoly/__init__.py:55`` but absent from the reference tree, so this file is the
oracle contract for the end-to-end path.  Every decision follows SURVEY.md
Appendix A, which cites SPEC.md:429-502 and PAPER.md:724-840:

* A.1 ``logm``          -- PAPER.md:724-749 (Algorithm 1)
* A.2 ``alpha``         -- PAPER.md:762-788 (Eqs. 24, 27, 28)
* A.3 ``select_order``  -- PAPER.md:790-836 (Eqs. 29-34, tabmin_im)

The driver is written against a pluggable primitive set ``prims``:
``OraclePrims`` (this package's numpy restatement, with margin tracking) or, in
``tests/golden/make_golden.py`` only, an adapter over the reference's own
primitives loaded from /root/reference.  Running the same driver over both and
comparing the outputs bit-for-bit is what pins the restated primitives.

Status codes (shared with the CUDA report, include/logmpoly_b200.h):
0 OK, 1 SINGULAR, 2 DB_NOCONV, 3 SCALING_MAXITER, 4 NONFINITE.
"""
import math

import numpy as np

from paper_2401_10089_b200 import constants as _C  # frozen data only (no product code)

from . import primitives as P

K_MAX = _C.K_MAX
K_DEFAULT = getattr(_C, "K_DEFAULT", _C.K_MAX)  # reference default (shipped schemes k <= 5)
THETA = _C.THETA
ORDER = _C.ORDER
TABMIN_IM = _C.TABMIN_IM

OK, SINGULAR, DB_NOCONV, SCALING_MAXITER, NONFINITE = 0, 1, 2, 3, 4


class OraclePrims:
    """The restated primitives (oracle/primitives.py) with margin tracking."""

    def __init__(self, schemes):
        self.schemes = schemes
        self.margins = P.Margins()

    def balance(self, A):
        return P.balance(A, margins=self.margins)

    def onenorm(self, A):
        return P.onenorm(A)

    def est_power_norm(self, M, p, counter):
        return P.est_power_norm(M, p, counter=counter, margins=self.margins)

    def est_product_norm(self, factors, counter):
        return P.est_product_norm(factors, counter=counter, margins=self.margins)

    def sqrt_db(self, A, counter):
        return P.sqrt_db(A, counter=counter, margins=self.margins)

    def matmul(self, A, B, counter):
        counter.products += 1
        return A @ B

    def eval_degopt(self, k, X, counter, first_product):
        return P.eval_degopt(self.schemes[k - 1], X, counter=counter, first_product=first_product)

    def note(self, x, thr):
        self.margins.cmp(x, thr)

    def min_margin(self):
        return self.margins.min_margin


class _State:
    """Per-call mutable state: counters, estimate cache, report fields."""

    def __init__(self, prims, theta, order, max_k):
        self.prims = prims
        self.theta = theta
        self.order = order
        self.K = max_k
        self.counter = P.Counter()
        self.cache = {}
        self.norm_estimations = 0
        self.s = 0
        self.db_iters = 0
        self.alpha_used = 0.0

    def note(self, x, thr):
        if hasattr(self.prims, "note"):
            self.prims.note(x, thr)

    def le(self, x, thr):
        self.note(x, thr)
        return x <= thr


def _alpha(st, AmI, AI2, nA, m, theta):
    """A.2: alpha_m ~ max(||(A-I)^m||^(1/m), ||(A-I)^(m+1)||^(1/(m+1))) with the
    Eq. 27 / Eq. 28 skips."""
    pr = st.prims
    if AI2 is not None:
        nI2 = pr.onenorm(AI2)
        r2 = math.sqrt(nI2)
        if st.le(r2, theta):                      # Eq. 27
            t1, Pm = r2, _pow(nI2, m // 2)
        else:
            if m not in st.cache:
                st.norm_estimations += 1
                st.cache[m] = pr.est_power_norm(AI2, m // 2, st.counter)
            Pm = st.cache[m]
            t1 = _pow(Pm, 1.0 / m)
    else:
        if m not in st.cache:
            st.norm_estimations += 1
            st.cache[m] = pr.est_power_norm(AmI, m, st.counter)
        Pm = st.cache[m]
        t1 = _pow(Pm, 1.0 / m)
    st.note(t1, theta)
    if t1 > theta:
        return t1
    bound = _pow(Pm * nA, 1.0 / (m + 1))               # Eq. 28
    if st.le(bound, theta):
        t2 = bound
    else:
        if (m + 1) not in st.cache:
            st.norm_estimations += 1
            if AI2 is not None:
                st.cache[m + 1] = pr.est_product_norm([(AI2, m // 2), (AmI, 1)], st.counter)
            else:
                st.cache[m + 1] = pr.est_power_norm(AmI, m + 1, st.counter)
        t2 = _pow(st.cache[m + 1], 1.0 / (m + 1))
    return max(t1, t2)


def _first_index(st, x):
    """min{j in 1..K : x <= Theta_j}, K if none (Eqs. 29-31)."""
    for j in range(1, st.K + 1):
        if st.le(x, st.theta[j - 1]):
            return j
    return st.K


def _select(st, AmI, AI2, nA, alpha_loop):
    """A.3 select_order.  Returns (k, alpha certifying k)."""
    K, th, mk = st.K, st.theta, st.order
    nI2 = st.prims.onenorm(AI2)
    r2 = math.sqrt(nI2)
    mK = mk[K - 1]
    # 1. min_im (Eqs. 29-31)
    if mK in st.cache:
        min_im = _first_index(st, _pow(st.cache[mK], 1.0 / mK))
        if (mK + 1) in st.cache:
            min_im = max(min_im, _first_index(st, _pow(st.cache[mK + 1], 1.0 / (mK + 1))))
    else:
        min_im = _first_index(st, r2)
    # 2. tabmin_im
    min_im = TABMIN_IM[min_im - 1]
    # 3.
    st.note(r2, th[0])
    min_im = max(min_im, 2) if r2 > th[0] else 1
    # 4. max_in (Eq. 32, all m_j even)
    max_in, max_bound = K, None
    for j in range(1, K + 1):
        m = mk[j - 1]
        b = _pow(_pow(nI2, m // 2) * nA, 1.0 / (m + 1))
        if st.le(b, th[j - 1]):
            max_in, max_bound = j, b
            break
    cert_max = max_bound if max_bound is not None else alpha_loop
    # 5.
    if min_im >= max_in:
        return max_in, cert_max
    # 6. sweep with the j+1 shortcut
    for j in range(min_im, max_in):
        a = _alpha(st, AmI, AI2, nA, mk[j - 1], th[j - 1])
        if st.le(a, th[j - 1]):
            return j, a
        if st.le(a, th[j]):
            return j + 1, a
    return max_in, cert_max


def _pow(x, y):
    """x ** y with IEEE overflow to inf (float64 semantics, like the GPU's pow) instead of
    Python's OverflowError: reachable only when the estimator itself overflowed (norms beyond
    ~1e300), where Algorithm 1's decisions are meaningless and the result is reported as
    non-finite."""
    with np.errstate(over="ignore", invalid="ignore"):
        return float(np.power(np.float64(x), np.float64(y)))


def _report(st, status, k=0, balanced=True, sweeps=0, msg=""):
    return {
        "status": status, "s": st.s, "k": k, "alpha_used": st.alpha_used,
        "db_iters": st.db_iters, "products": st.counter.products,
        "divisions": st.counter.divisions, "estimation_passes": st.counter.estimation_passes,
        "norm_estimations": st.norm_estimations, "balanced": bool(balanced),
        "balance_sweeps": sweeps,
        "min_margin": st.prims.min_margin() if hasattr(st.prims, "min_margin") else math.nan,
        "db_plateau": st.prims.margins.db_plateau if hasattr(st.prims, "margins") else 0,
        "message": msg,
    }


def logm_status(A, prims, theta=THETA, order=ORDER, max_k=K_DEFAULT, maxiter=40, do_balance=True):
    """Algorithm 1 (A.1).  Returns (L or None, report dict); never raises for numerical
    failures -- the status code carries them (mirrors the GPU report)."""
    st = _State(prims, theta, order, max_k)
    K = max_k
    try:
        A = P.as_square(A)
    except ValueError as exc:
        return None, _report(st, NONFINITE, msg=str(exc))
    n = A.shape[0]
    I = np.eye(n)
    sweeps = 0
    if do_balance:
        B, scale, sweeps = prims.balance(A)
    else:
        B, scale = A.copy(), np.ones(n)
    thK = theta[K - 1]
    AI2 = None
    alpha_loop = prims.onenorm(B - I)
    finish = st.le(alpha_loop, thK)
    try:
        while not finish and st.s < maxiter:
            AmI = B - I
            nA = prims.onenorm(AmI)
            a = _alpha(st, AmI, AI2, nA, order[K - 1], thK)
            alpha_loop = a
            finish = st.le(a, thK)
            if not finish:
                Aprev = B
                B, its = prims.sqrt_db(B, st.counter)
                st.db_iters += its
                st.s += 1
                AI2 = Aprev - 2 * B + I
                st.cache = {}
    except Exception as exc:        # noqa: BLE001 -- classify like the GPU status codes
        name = type(exc).__name__
        if name == "SingularMatrixError":
            code = SINGULAR
        elif name == "ConvergenceError":
            code = DB_NOCONV
        elif isinstance(exc, ValueError):
            code = NONFINITE
        else:
            raise
        # iterations spent inside the failing root: two divisions per DB iteration
        st.db_iters = st.counter.divisions // 2
        return None, _report(st, code, balanced=do_balance, sweeps=sweeps, msg=str(exc))
    if not finish:
        return None, _report(st, SCALING_MAXITER, balanced=do_balance, sweeps=sweeps,
                             msg=f"no convergence after {maxiter} square roots")
    AmI = B - I
    nA = prims.onenorm(AmI)
    if AI2 is None:
        AI2 = prims.matmul(AmI, AmI, st.counter)
    k, cert = _select(st, AmI, AI2, nA, alpha_loop)
    st.alpha_used = cert
    Z = prims.eval_degopt(k, I - B, st.counter, AI2)
    with np.errstate(over="ignore", invalid="ignore"):
        L = -(2.0 ** st.s) * Z
        if do_balance:
            L = P.unbalance(L, scale)
    if not np.all(np.isfinite(L)):  # overflow inside the polynomial (estimator overflow upstream)
        return L, _report(st, NONFINITE, k=k, balanced=do_balance, sweeps=sweeps, msg="non-finite result")
    return L, _report(st, OK, k=k, balanced=do_balance, sweeps=sweeps)


def default_prims():
    return OraclePrims(_C.SCHEMES)


def logm(A, **kw):
    """Convenience: restated logm over the restated primitives; raises on failure."""
    L, rep = logm_status(A, default_prims(), **kw)
    if rep["status"] == SINGULAR:
        raise P.SingularMatrixError(rep["message"])
    if rep["status"] in (DB_NOCONV, SCALING_MAXITER):
        raise P.ConvergenceError(rep["message"], rep)
    if rep["status"] == NONFINITE:
        raise ValueError(rep["message"])
    return L, rep
