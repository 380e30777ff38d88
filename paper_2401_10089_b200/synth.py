"""Seeded synthetic matrix families for the five BASELINE.json configs (+ variants 3b/5b).

The paper's own test sets are not in this container; these
generators stand in for them with the shapes, sizes and value distributions that
BASELINE.json names.  All generation is float64 numpy on
the CPU with ``numpy.random.default_rng``, so the oracle and the GPU see the same
bits.  ``config(c, batch=None, n=None, seed=None)`` returns a (B, n, n) C-order array.
"""
import numpy as np

# (name, n, batch) as in BASELINE.json "configs"
CONFIGS = {
    1: ("spd64", 64, 1),
    2: ("near_identity32", 32, 4096),
    3: ("nonnormal128", 128, 1024),
    4: ("spd512", 512, 256),
    5: ("nonnormal4096", 4096, 8),
    "3b": ("nonnormal128_wellcond", 128, 1024),
    "5b": ("nonnormal4096_wellcond", 4096, 8),
}

SEEDS = {1: 0, 2: 2, 3: 3, 4: 4, 5: 5, "3b": 31, "5b": 51}


def _haar(rng, n):
    G = rng.standard_normal((n, n))
    Q, R = np.linalg.qr(G)
    return Q * np.sign(np.diag(R))[None, :]


def spd(rng, n, lo, hi, haar=True):
    """A = Q diag(lambda) Q^T, lambda log-uniform in [10^lo, 10^hi]."""
    if haar:
        Q = _haar(rng, n)
    else:
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = 10.0 ** rng.uniform(lo, hi, n)
    A = (Q * lam[None, :]) @ Q.T
    return 0.5 * (A + A.T)


def near_identity(rng, n):
    """A = I + 0.9 G / ||G||_2, G i.i.d. N(0, 1)."""
    G = rng.standard_normal((n, n))
    return np.eye(n) + 0.9 * G / np.linalg.norm(G, 2)


def nonnormal(rng, n, lo, hi, wellcond=False):
    """A = S T S^-1 with T upper triangular, diag log-uniform in [10^lo, 10^hi].

    As written (BASELINE.json configs 3 and 5): strict upper N(0, 0.1^2),
    S = I + 0.1 N(0, 1).  ``wellcond`` gives the labelled supplementary variant
    (3b/5b): T = D (I + N) with N strict upper N(0, (0.1/sqrt n)^2),
    S = I + 0.1 G / sqrt(n).
    """
    d = 10.0 ** rng.uniform(lo, hi, n)
    if wellcond:
        N = np.triu(rng.standard_normal((n, n)) * (0.1 / np.sqrt(n)), 1)
        T = d[:, None] * (np.eye(n) + N)
        S = np.eye(n) + 0.1 * rng.standard_normal((n, n)) / np.sqrt(n)
    else:
        T = np.triu(rng.standard_normal((n, n)) * 0.1, 1) + np.diag(d)
        S = np.eye(n) + 0.1 * rng.standard_normal((n, n))
    return np.linalg.solve(S.T, (S @ T).T).T       # S T S^-1


def config(c, batch=None, n=None, seed=None):
    """Batch of matrices for config ``c`` (1..5, "3b", "5b")."""
    name, n0, b0 = CONFIGS[c]
    n = n0 if n is None else n
    batch = b0 if batch is None else batch
    seed = SEEDS[c] if seed is None else seed
    rng = np.random.default_rng(seed)
    out = np.empty((batch, n, n))
    for b in range(batch):
        if c == 1:
            out[b] = spd(rng, n, -2.0, 2.0, haar=False)
        elif c == 2:
            out[b] = near_identity(rng, n)
        elif c == 3:
            out[b] = nonnormal(rng, n, -3.0, 3.0)
        elif c == "3b":
            out[b] = nonnormal(rng, n, -3.0, 3.0, wellcond=True)
        elif c == 4:
            out[b] = spd(rng, n, -4.0, 4.0)
        elif c == 5:
            out[b] = nonnormal(rng, n, -2.0, 2.0)
        elif c == "5b":
            out[b] = nonnormal(rng, n, -2.0, 2.0, wellcond=True)
        else:
            raise ValueError(f"unknown config {c!r}")
    return out


def known_log(rng, n, kappa=10.0):
    """A = V diag(e^lambda) V^-1 with its exact log V diag(lambda) V^-1.

    Real spectrum lambda in [-1, 1]; V = U diag(sv) W^T with singular values
    log-spaced in [1, kappa] (so cond_2(V) = kappa).
    """
    U = _haar(rng, n)
    W = _haar(rng, n)
    sv = np.logspace(0.0, np.log10(kappa), n)
    V = (U * sv[None, :]) @ W.T
    lam = rng.uniform(-1.0, 1.0, n)
    Vi = np.linalg.inv(V)
    A = (V * np.exp(lam)[None, :]) @ Vi
    L = (V * lam[None, :]) @ Vi
    return A, L
