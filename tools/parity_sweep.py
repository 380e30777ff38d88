"""Randomized parity sweep: GPU logm vs the CPU oracle over many sizes / families / seeds.

    python tools/parity_sweep.py [--count 600] [--nmax 160 | --sizes 320,384,448,512] [--seed 0] [--workers 16]

Families: near-identity (config 2 style), SPD with a wide spectrum, non-normal (3b style),
known-log.  For each matrix: status / s / k / db_iters / counters classified as in
tests/parity.py (match / exempt / db_plateau / mismatch) and, when statuses are OK and
(s, k) agree, the L error against the oracle's tolerance.  Prints a JSON summary and the
worst cases; exit code 1 on any mismatch or tolerance failure.  Test infrastructure: uses
the oracle (tests/, smoke() and bench.py's CPU legs are the other users).
"""
import argparse
import json
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _oracle(A):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    from oracle import driver as D
    L, rep = D.logm_status(A, D.default_prims())
    return L, rep


def make(rng, fam, n):
    from paper_2401_10089_b200 import synth
    if fam == "scaled":        # huge / tiny magnitudes (balancing, many square roots)
        return synth.near_identity(rng, n) * 10.0 ** rng.uniform(-60, 60)
    if fam == "illcond":       # SPD with kappa up to 1e12
        return synth.spd(rng, n, -6.0, 6.0)
    if fam == "bignorm":       # needs many square roots
        return synth.spd(rng, n, 2.0, 8.0)
    if fam == "jordanish":     # identity + strong nilpotent part
        return np.eye(n) + np.triu(rng.standard_normal((n, n)) * 3.0, 1)
    if fam == "negdiag":       # an eigenvalue on the negative real axis: DB non-convergence
        d = 10.0 ** rng.uniform(-1, 1, n)
        d[int(rng.integers(0, n))] *= -1.0
        return np.diag(d)
    if fam == "rotation":      # eigenvalues on the unit circle (principal log exists if no -1)
        th = rng.uniform(-3.0, 3.0, n // 2)
        R = np.eye(n)
        for q, t in enumerate(th):
            c, s_ = np.cos(t), np.sin(t)
            R[2 * q:2 * q + 2, 2 * q:2 * q + 2] = [[c, -s_], [s_, c]]
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        return Q @ R @ Q.T
    if fam == "near":
        return synth.near_identity(rng, n)
    if fam == "spd":
        return synth.spd(rng, n, -3.0, 3.0)
    if fam == "nonnormal":
        return synth.nonnormal(rng, n, -2.0, 2.0, wellcond=True)
    A, _ = synth.known_log(rng, n, kappa=float(10.0 ** rng.uniform(0, 2)))
    return A


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--count", type=int, default=600)
    ap.add_argument("--nmax", type=int, default=160)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--sizes", default=None, help="comma-separated n to draw from (default 1..nmax)")
    ap.add_argument("--workers", type=int, default=min(16, os.cpu_count() or 1))
    ap.add_argument("--extreme", action="store_true", help="scaled / ill-conditioned / big-norm / "
                    "Jordan-like / negative-eigenvalue / rotation families")
    args = ap.parse_args()
    import paper_2401_10089_b200 as lp
    from tests.parity import classify, rel_err, tolerance
    rng = np.random.default_rng(args.seed)
    fams = (["scaled", "illcond", "bignorm", "jordanish", "negdiag", "rotation"] if args.extreme
            else ["near", "spd", "nonnormal", "knownlog"])
    sizes = [int(x) for x in args.sizes.split(",")] if args.sizes else None
    cases = []
    for q in range(args.count):
        n = int(rng.choice(sizes)) if sizes else int(rng.integers(1, args.nmax + 1))
        fam = fams[q % len(fams)]
        cases.append((q, fam, n, make(rng, fam, n)))
    # GPU: group by n
    gpu = {}
    for n in sorted({c[2] for c in cases}):
        grp = [c for c in cases if c[2] == n]
        L, reps = lp.logm_batched(np.stack([c[3] for c in grp]), lp.LogmOptions(raise_on_error=False))
        for c, Lg, r in zip(grp, np.asarray(L), reps):
            gpu[c[0]] = (Lg, r)
    with mp.get_context("spawn").Pool(args.workers) as pool:
        orc = pool.map(_oracle, [c[3] for c in cases], chunksize=4)
    counts = {"match": 0, "exempt": 0, "db_plateau": 0, "mismatch": 0}
    bad, worst = [], []
    for c, (Lo, ro) in zip(cases, orc):
        Lg, rg = gpu[c[0]]
        cls, g, o = classify(rg, ro)
        counts[cls] += 1
        if cls == "mismatch":
            bad.append({"id": c[0], "fam": c[1], "n": c[2], "gpu": g, "oracle": o})
            continue
        if g["status"] == 0 and o["status"] == 0 and (g["s"], g["k"]) == (o["s"], o["k"]) and \
                np.isfinite(Lo).all():
            e, tol = rel_err(Lg, Lo), tolerance(c[3], Lo)
            worst.append((e / tol, c[0], c[1], c[2], e, tol))
            if e > tol:
                bad.append({"id": c[0], "fam": c[1], "n": c[2], "err": e, "tol": tol})
    worst.sort(reverse=True)
    print(json.dumps({"cases": len(cases), "classes": counts, "failures": len(bad),
                      "worst_err_over_tol": [list(w) for w in worst[:5]]}, indent=1))
    for b in bad[:20]:
        print("FAIL", b)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
