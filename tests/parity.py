"""Parity bookkeeping shared by the GPU tests and bench.py's parity summary.

A GPU report agrees with the oracle when status, s, k, db_iters (and the counters derived
from them) are equal.  Following SURVEY.md 8(d), a disagreement is *exempt* only when
either side recorded a decision within 1e-10 (relative) of its threshold; the DB stopping
test ``rel <= 10 n u`` compares a quantity that is itself rounding noise at convergence,
so it is reported separately (``db_plateau``) when the only difference is the iteration
count of an ill-conditioned root.
"""
import numpy as np

FIELDS = ("status", "s", "k", "db_iters", "products", "divisions", "estimation_passes",
          "norm_estimations")
EXEMPT_MARGIN = 1e-10


def gpu_fields(rec):
    return {f: int(rec[f]) for f in FIELDS}


def classify(gpu_rec, oracle_rep):
    g = gpu_fields(gpu_rec)
    o = {f: int(oracle_rep[f]) for f in FIELDS}
    if g == o:
        return "match", g, o
    m = min(float(gpu_rec["min_margin"]), float(oracle_rep["min_margin"]))
    if m < EXEMPT_MARGIN:
        return "exempt", g, o
    if int(gpu_rec["db_plateau"]) > 0 or int(oracle_rep.get("db_plateau", 0)) > 0:
        return "db_plateau", g, o
    return "mismatch", g, o


def rel_err(L, Lref):
    den = np.linalg.norm(Lref)
    return np.linalg.norm(L - Lref) / (den if den > 0 else 1.0)


def tolerance(A, Lref):
    """1e-12 on well-conditioned cases, else 10 cond_log u with cond_log estimated by
    kappa_2(A) ||A||_F / ||log A||_F (exact 1/lambda_min form for SPD)."""
    u = 2.0 ** -53
    nl = np.linalg.norm(Lref)
    if nl == 0:
        return 1e-12
    if np.array_equal(A, A.T):
        w = np.linalg.eigvalsh(A)
        cond = np.linalg.norm(A) / (w.min() * nl) if w.min() > 0 else np.inf
    else:
        cond = np.linalg.cond(A) * np.linalg.norm(A) / nl
    return max(1e-12, 10.0 * cond * u)
