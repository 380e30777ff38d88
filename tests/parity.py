"""Parity bookkeeping shared by the GPU tests, tools/parity_sweep.py and bench.py.

A GPU report agrees with the oracle when status, s, k, db_iters (and the counters derived
from them) are equal.  Following SURVEY.md 8(d), a disagreement is *exempt* only when
either side recorded a decision within 1e-10 (relative) of its threshold.

``db_plateau``: the DB stopping test ``rel <= 10 n u`` (sqrtm.py:44-45, 74) compares a
quantity that is itself rounding noise at convergence, so the iteration count of an
ill-conditioned root is not reproducible by different (equally accurate) arithmetic.  Such a
record is classified ``db_plateau`` only when status, s, k, products and norm_estimations
are all equal and the only differences are db_iters and the counters derived from it
(divisions = 2 db_iters, and estimation_passes of the estimates taken on the slightly
different square roots), and either side recorded a stop test with rel within a factor 10
of tol.  The caller still checks L against the accuracy tolerance for it.  Any other
difference -- a different status, s or k -- is a ``mismatch`` unless the margin exemption
applies.

``db_stall``: the noise floor itself.  On kappa ~ 1e8 inputs at small n, rel/tol settles at
O(1) rounding noise (e.g. 1.03 .. 1.99 for 40 iterations) and whether it ever dips below 1
before the 50-iteration cap depends on the inversion's rounding: the oracle (LAPACK
getrf/getrs) stalls on some matrices where Gauss-Jordan converges and vice versa.  A record
is ``db_stall`` only when one side is DB_NOCONV after >= 10 plateau stop tests (it sat at the
noise floor, never within reach of the scaling decisions) and the other side converged after
at least one plateau stop test.  Tests state how many they allow (0 on the BASELINE configs).
"""
import multiprocessing as mp
import os

import numpy as np

FIELDS = ("status", "s", "k", "db_iters", "products", "divisions", "estimation_passes",
          "norm_estimations")
# fields a db_plateau record may differ in (everything else must be equal)
PLATEAU_FREE = ("db_iters", "divisions", "estimation_passes")
EXEMPT_MARGIN = 1e-10
STALL_PLATEAU = 10


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
    gp, op = int(gpu_rec["db_plateau"]), int(oracle_rep.get("db_plateau", 0))
    if (gp > 0 or op > 0) and all(g[f] == o[f] for f in FIELDS if f not in PLATEAU_FREE):
        return "db_plateau", g, o
    if {g["status"], o["status"]} == {0, 2}:
        stalled, conv = (gp, op) if g["status"] == 2 else (op, gp)
        if stalled >= STALL_PLATEAU and conv >= 1:
            return "db_stall", g, o
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


# ------------------------------------------------------------------ oracle over many cores

def _oracle_init(threads):
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    import sys
    if root not in sys.path:
        sys.path.insert(0, root)


def _oracle_one(A, max_k=None):
    from oracle import driver as D
    kw = {} if max_k is None else {"max_k": max_k}
    L, rep = D.logm_status(A, D.default_prims(), **kw)
    rep = {k: v for k, v in rep.items() if k != "message"}
    return L, rep


def _oracle_check_one(args):
    """Worker: oracle on one matrix, then the accuracy check against the GPU result (so the
    n x n L never travels back to the parent)."""
    A, Lg, max_k = args
    Lr, rr = _oracle_one(A, max_k)
    err = tol = None
    if Lr is not None and Lg is not None:
        err, tol = rel_err(Lg, Lr), tolerance(A, Lr)
    return rr, err, tol


def oracle_reports(As, Ls, reps, procs=None, max_k=None):
    """Run the oracle on every matrix of As (process pool, one BLAS thread per worker; a
    single matrix runs in-process with all-core BLAS) and return, per matrix, (oracle report,
    rel error of the GPU L, tolerance)."""
    B = As.shape[0]
    items = [(As[b], None if Ls is None else np.asarray(Ls[b]), max_k) for b in range(B)]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    procs = procs or min(cores, B)
    if B == 1 or procs == 1:
        return [_oracle_check_one(it) for it in items]
    ctx = mp.get_context("spawn")
    with ctx.Pool(procs, initializer=_oracle_init, initargs=(max(1, cores // procs),)) as pool:
        return pool.map(_oracle_check_one, items, chunksize=max(1, B // (4 * procs)))


def check_batch(As, L, reps, allow_mismatch=0, procs=None, verbose=True, allow_stall=0, max_k=None):
    """Compare GPU (L, reports) with the oracle per matrix.  match / db_plateau records with
    status OK on both sides must meet the L tolerance; mismatches are counted (<= allowed).
    An exempt record with equal (status, s, k) is held to the L tolerance as well."""
    counts = {"match": 0, "exempt": 0, "db_plateau": 0, "db_stall": 0, "mismatch": 0}
    worst = 0.0
    res = oracle_reports(As, L, reps, procs, max_k)
    for b, (rr, err, tol) in enumerate(res):
        cls, g, o = classify(reps[b], rr)
        counts[cls] += 1
        if cls in ("mismatch", "db_stall") and verbose:
            print(cls.upper(), b, "gpu", g, "oracle", o, "margins", float(reps[b]["min_margin"]), rr["min_margin"])
        both_ok = rr["status"] == 0 and int(reps[b]["status"]) == 0
        same = (g["status"], g["s"], g["k"]) == (o["status"], o["s"], o["k"])
        if both_ok and same and cls != "mismatch":
            assert err is not None
            worst = max(worst, err / tol)
            assert err <= tol, (b, cls, err, tol)
    if verbose:
        print(counts, "worst err/tol", worst)
    assert counts["mismatch"] <= allow_mismatch, counts
    assert counts["db_stall"] <= allow_stall, counts
    return counts, res
