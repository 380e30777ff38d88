import sys, numpy as np
sys.path.insert(0, '.')
import paper_2401_10089_b200 as lp
from oracle import primitives as P
for n in [520, 544, 576, 1000, 2048]:
    rng = np.random.default_rng(n)
    G = rng.standard_normal((1, n, n))
    A = np.eye(n)[None] + 0.5 * G / np.linalg.norm(G[0], 2)
    X, its, st = lp.sqrt_db_batched(A)
    msg = ""
    if n <= 1000:
        Xo, ito = P.sqrt_db(A[0]); msg = f"oracle its {ito} err {np.linalg.norm(X[0]-Xo)/np.linalg.norm(Xo):.2e}"
    print(n, "status", st, "its", its, "finite", np.isfinite(X).all(), msg, flush=True)
