"""Evidence for the db_stall parity class (tests/parity.py): the oracle's DB relative change
rel / tol per iteration on the config-4-shaped matrices where it differs from the GPU, and
the oracle's outcome under 1-ulp perturbations of A.

    python tools/db_stall_evidence.py > profiles/r02/db_stall_evidence.txt
"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import driver as D  # noqa: E402
from oracle import primitives as P  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402


def trace(A):
    n = A.shape[0]
    tol = 10 * n * 2.0 ** -53
    X, Y, scaling, rels = A.copy(), np.eye(n), True, []
    for it in range(1, 51):
        fx, lx = P.lu_logabsdet(X)
        fy, ly = P.lu_logabsdet(Y)
        mu = min(max(math.exp(-(lx + ly) / (2 * n)), 1e-8), 1e8) if scaling else 1.0
        Xi, Yi = P.lu_inverse(fx), P.lu_inverse(fy)
        Xn, Yn = 0.5 * (mu * X + Yi / mu), 0.5 * (mu * Y + Xi / mu)
        rel = P.onenorm(Xn - X) / P.onenorm(Xn)
        X, Y = Xn, Yn
        if rel < 1e-2:
            scaling = False
        rels.append(rel / tol)
        if rel <= tol:
            break
    return it, rels


for (n, B, idx) in [(48, 16, 4), (80, 4, 2)]:
    A = synth.config(4, batch=B, n=n)[idx]
    w = np.linalg.eigvalsh(A)
    it, rels = trace(A)
    print(f"config-4 spectrum, n = {n}, matrix {idx} of synth.config(4, batch={B}, n={n}); kappa_2 = {w.max() / w.min():.3g}")
    print(f"  oracle first root: {it} DB iterations; rel / tol from iteration 6: " + " ".join(f"{r:.2f}" for r in rels[5:]))
    outs = []
    for t in range(6):
        Ap = A.copy()
        if t:
            rng = np.random.default_rng(t)
            Ap = Ap * (1 + rng.choice([-1, 1], size=A.shape) * 2.0 ** -52)
            Ap = 0.5 * (Ap + Ap.T)
        _, r = D.logm_status(Ap, D.default_prims())
        outs.append((r["status"], r["s"], r["db_iters"]))
    print("  oracle (status, s, db_iters) for A and 5 perturbations by 1 ulp: " + str(outs))
