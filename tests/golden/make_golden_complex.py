"""Golden vectors for the complex128 branch of the oracle, written by the reference's own
primitives (run in the build container only: needs /root/reference).

    python tests/golden/make_golden_complex.py

The reference accepts complex input (as_square, matcore.py:60-61) and estimates with the
complex sign (matcore.py:226-231).  This runs the restated driver (oracle/driver.py) over the
reference primitives (the RefPrims adapter of make_golden.py) on complex matrices and stores
L and the report integers, plus primitive outputs (est_power_norm, sqrt_db, balance) on
complex inputs; tests/test_oracle_golden.py requires the restatement to reproduce them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, ROOT)
from make_golden import RefPrims, load_reference  # noqa: E402

FIELDS = ("status", "s", "k", "db_iters", "products", "divisions", "estimation_passes", "norm_estimations")


def cases():
    rng = np.random.default_rng(20260120)
    out = []
    for n, scale in ((1, 0.5), (3, 0.3), (8, 0.9), (16, 0.6), (24, 2.0), (40, 0.95)):
        G = (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(2 * n)
        out.append((f"nearI_{n}", np.eye(n) + scale * G / max(np.linalg.norm(G, 2), 1e-300)))
    # Hermitian positive definite with a wide spectrum, badly scaled copy (balancing acts)
    n = 20
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n)))
    lam = 10.0 ** rng.uniform(-2, 2, n)
    H = (Q * lam) @ Q.conj().T
    out.append(("hpd20", 0.5 * (H + H.conj().T)))
    d = 2.0 ** rng.integers(-12, 12, n)
    out.append(("hpd20_scaled", out[-1][1] * (d[:, None] / d[None, :])))
    # complex-spectrum rotation (eigenvalues e^{+-i 0.7} etc.) and a negative real eigenvalue
    out.append(("rot2c", np.array([[np.cos(0.7), -np.sin(0.7)], [np.sin(0.7), np.cos(0.7)]]) * (1 + 0.5j)))
    out.append(("negreal3", np.diag([-2.0 + 0j, 1.0, 3.0j])))
    # nonnormal S T S^-1 with a complex log-uniform spectrum at n = 128 (several square roots;
    # pins the restated sqrt_db's complex identity at sizes where numpy's result layout changes)
    n = 128
    mag = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
    ph = rng.uniform(-2.5, 2.5, n)
    T = np.diag(mag * np.exp(1j * ph)) + np.triu((0.3 / n) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))), 1)
    S = np.eye(n) + 0.1 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
    out.append(("nonnormal128", S @ T @ np.linalg.inv(S)))
    return out


def main():
    mc, sc, sq = load_reference()
    from oracle import driver as D
    prims = RefPrims(mc, sc, sq)
    out, names = {}, []
    for name, A in cases():
        L, rep = D.logm_status(A, prims)
        names.append(name)
        out[f"drv/{name}/A"] = A
        out[f"drv/{name}/L"] = L if L is not None else np.zeros((0, 0), dtype=np.complex128)
        out[f"drv/{name}/ints"] = np.array([rep[f] for f in FIELDS], dtype=np.int64)
        print(f"{name:14s} n={A.shape[0]:3d} " + " ".join(f"{f}={rep[f]}" for f in FIELDS))
    rng = np.random.default_rng(7)
    M = (rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12))) / 4
    for p in (1, 3, 8):
        c = mc.OpCounter()
        out[f"prim/est/{p}"] = np.array([mc.est_power_norm(M, p, counter=c), c.estimation_passes])
    out["prim/est/M"] = M
    S = np.eye(12) + 0.4 * M
    out["prim/sqrt/A"] = S
    out["prim/sqrt/X"] = sq.sqrt_db(S)
    Bb, T = mc.balance(M * (2.0 ** np.arange(12))[:, None])
    out["prim/bal/A"] = M * (2.0 ** np.arange(12))[:, None]
    out["prim/bal/B"] = Bb
    out["prim/bal/scale"] = T.scale
    out["drv_names"] = np.array(names)
    out["drv_fields"] = np.array(FIELDS)
    path = os.path.join(HERE, "golden_complex_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
