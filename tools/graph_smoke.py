"""Quick Engine G graph smoke (diagnostics): sqrt_db / estimate / logm at a few n with the
capture trace on (LGM_GRAPH_DEBUG=1), each compared with the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_10089_b200 as lp  # noqa: E402
from oracle import primitives as P  # noqa: E402
from oracle import driver as D  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402

for n in [int(x) for x in (sys.argv[1:] or ["65", "130", "320"])]:
    rng = np.random.default_rng(n)
    G = rng.standard_normal((2, n, n))
    A = np.eye(n)[None] + 0.5 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    X, its, st = lp.sqrt_db_batched(A)
    Xo, ito = P.sqrt_db(A[0])
    print("sqrt_db", n, list(its), list(st), "oracle its", ito, "err", np.linalg.norm(X[0] - Xo) / np.linalg.norm(Xo), flush=True)
    As = synth.config("3b", batch=3, n=n)
    L, reps = lp.logm_batched(As, lp.LogmOptions(raise_on_error=False))
    for b in range(3):
        Lr, rr = D.logm_status(As[b], D.default_prims())
        print("logm", n, b, {f: int(reps[b][f]) for f in ("status", "s", "k", "db_iters", "estimation_passes")},
              {f: rr[f] for f in ("status", "s", "k", "db_iters", "estimation_passes")},
              "err", np.linalg.norm(L[b] - Lr) / np.linalg.norm(Lr) if Lr is not None else None, flush=True)
print("graph smoke done")
