"""Tiny workload that launches every kernel of the library once or a few times, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py [--quick]

Engine F (n = 32 full, 48 partial, 64 full), Engine G: G1 (n = 100, odd n = 101 with the
fused-left-operand GEMM), G2 single-CTA panels + rank-64 passes (n = 320), G2 cluster panels
(n = 576, skipped with --quick), the estimator (fused and per-step kernels), balance, and the
building blocks sqrt_db / est / balance / eval_degopt on both engines.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402


def main():
    quick = "--quick" in sys.argv
    opts = lp.LogmOptions(raise_on_error=False)
    sizes = [(2, 32), ("3b", 48), (4, 64), ("3b", 100), (2, 101), (4, 320)]
    if not quick:
        sizes.append(("5b", 576))
    for c, n in sizes:
        A = synth.config(c, batch=2 if n <= 128 else 1, n=n)
        L, reps = lp.logm_batched(A, opts)
        print("logm", c, n, list(reps["status"]), list(reps["s"]), list(reps["k"]), flush=True)
    # failure paths: non-finite input, singular, DB no-convergence (NaN fill of L)
    bad = np.stack([np.full((80, 80), np.nan), np.diag(np.r_[-1.0, np.linspace(2, 3, 79)])])
    _, reps = lp.logm_batched(bad, opts)
    print("failures", list(reps["status"]), flush=True)
    for n in (32, 80):
        A = synth.config("3b", batch=2, n=n)
        X, its, st = lp.sqrt_db_batched(A)
        est, passes = lp.primitives._est(A, 3, None, 5, True)
        est2, _ = lp.primitives._est(A, 2, A, 5, False)
        B, sc, sw = lp.balance_batched(A)
        Z = lp.eval_degopt(3, 0.1 * (A - np.eye(n)))
        print("blocks", n, list(st), list(passes), list(sw), float(np.abs(Z).max()), flush=True)
    print("sanitize probe done")


if __name__ == "__main__":
    main()
