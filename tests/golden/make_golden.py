"""Generate tests/golden/golden_v1.npz from the REFERENCE's own primitives.

Run in the build container only (needs /root/reference):
    python tests/golden/make_golden.py

The reference package cannot be imported normally (``logmpoly/__init__.py:55``
imports the missing ``logmpoly.driver``), so a stub package whose ``__path__``
points at /root/reference/pkg/src/logmpoly is registered first and the surviving
modules (matcore, sqrtm, schemes) are imported through it.

Two kinds of fixtures are written:

* ``prim/*``   -- reference primitive outputs on seeded inputs: ``balance``
  (matcore.py:180-215), ``onenorm`` (:84-87), ``est_power_norm`` /
  ``est_product_norm`` (:234-311, with OpCounter.estimation_passes), ``sqrt_db``
  (sqrtm.py:27-78, with OpCounter.divisions) and ``eval_degopt``
  (schemes.py:104-126) for the shipped schemes k = 1..5.
* ``drv/*``    -- the restated Algorithm 1 (oracle/driver.py) run over the
  reference primitives (``RefPrims`` below) on seeded inputs shaped like the
  BASELINE.json configs (small batches) plus SPEC edge cases.

``tests/test_oracle_golden.py`` checks the in-repo restatement (oracle/) against
these fixtures; the GPU parity tests use the same inputs.
"""
import os
import sys
import types

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src/logmpoly"


def load_reference():
    if "logmpoly" not in sys.modules:
        pkg = types.ModuleType("logmpoly")
        pkg.__path__ = [REF_SRC]
        sys.modules["logmpoly"] = pkg
    import logmpoly.matcore as mc
    import logmpoly.schemes as sc
    import logmpoly.sqrtm as sq
    return mc, sc, sq


class RefPrims:
    """oracle.driver primitive interface implemented by the reference's own functions."""

    def __init__(self, mc, sc, sq):
        self.mc, self.sc, self.sq = mc, sc, sq

    def _ctr(self):
        return self.mc.OpCounter()

    @staticmethod
    def _add(dst, src):
        dst.products += src.products
        dst.divisions += src.divisions
        dst.estimation_passes += src.estimation_passes

    def balance(self, A):
        B, T = self.mc.balance(A)
        return B, T.scale.copy(), -1

    def onenorm(self, A):
        return self.mc.onenorm(A)

    def est_power_norm(self, M, p, counter):
        c = self._ctr()
        try:
            return self.mc.est_power_norm(M, p, counter=c)
        finally:
            self._add(counter, c)

    def est_product_norm(self, factors, counter):
        c = self._ctr()
        try:
            return self.mc.est_product_norm(factors, counter=c)
        finally:
            self._add(counter, c)

    def sqrt_db(self, A, counter):
        c = self._ctr()
        try:
            X = self.sq.sqrt_db(A, counter=c)
        finally:
            self._add(counter, c)
        return X, c.divisions // 2

    def matmul(self, A, B, counter):
        c = self._ctr()
        out = self.mc.mat_mul(A, B, counter=c)
        self._add(counter, c)
        return out

    def eval_degopt(self, k, X, counter, first_product):
        c = self._ctr()
        out = self.sc.eval_degopt(self.sc.builtin_scheme(k), X, counter=c,
                                  first_product=first_product)
        self._add(counter, c)
        return out


def driver_cases():
    from paper_2401_10089_b200 import synth
    rng = np.random.default_rng(20240119)
    cases = []     # (name, A)
    cases.append(("cfg1", synth.config(1)[0]))
    for b, A in enumerate(synth.config(2, batch=24)):
        cases.append((f"cfg2_{b}", A))
    for b, A in enumerate(synth.config("3b", batch=6, n=32)):
        cases.append((f"cfg3b_n32_{b}", A))
    for b, A in enumerate(synth.config(4, batch=4, n=48)):
        cases.append((f"cfg4_n48_{b}", A))
    for b, A in enumerate(synth.config(3, batch=2, n=24)):
        cases.append((f"cfg3_n24_{b}", A))
    for n in (1, 2, 3, 5):
        cases.append((f"eye{n}", np.eye(n)))
    cases.append(("diag4", np.diag([4.0, 9.0, 0.25, 2.0])))
    cases.append(("scalar1", np.array([[7.5]])))
    cases.append(("scalar_near1", np.array([[1.0 + 1e-9]])))
    # near-identity spread exercising s = 0 and k = 1..5
    for e, eps in enumerate((1e-12, 1e-9, 1e-6, 1e-4, 3e-3, 2e-2, 8e-2, 0.2)):
        n = (7, 16, 24, 32, 13, 40, 33, 64)[e]
        G = rng.standard_normal((n, n))
        cases.append((f"nearI_{e}", np.eye(n) + eps * G / np.linalg.norm(G, 2)))
    for e in range(3):
        A, _ = synth.known_log(rng, (8, 16, 31)[e], kappa=10.0)
        cases.append((f"knownlog_{e}", A))
    # nonnormal Jordan-like: 0.3 (I + 5 superdiag) + I
    J = np.eye(4) + 0.3 * (np.eye(4) + 5.0 * np.eye(4, k=1))
    cases.append(("jordan4", J))
    # badly scaled: balancing must act (D A D^-1, D = 2^j)
    n = 20
    d = 2.0 ** rng.integers(-20, 20, n)
    A = synth.spd(rng, n, -1.0, 1.0)
    cases.append(("scaled20", A * (d[:, None] / d[None, :])))
    # failure statuses
    cases.append(("negeig3", np.diag([-1.0, 2.0, 3.0])))                       # DB no convergence
    Z = np.eye(4)
    Z[2, :] = 0.0
    cases.append(("singular4", Z))                                                # zero pivot
    return cases


def prim_cases(mc, sc, sq):
    rng = np.random.default_rng(7)
    out = {}
    # balance: badly scaled nonsymmetric matrices (includes n > 128: pairwise-sum branch)
    for n in (1, 5, 17, 32, 64, 130):
        d = 2.0 ** rng.integers(-30, 30, n)
        A = rng.standard_normal((n, n)) * (d[:, None] / d[None, :])
        if n > 3:
            A[1, 0] = 0.0
        B, T = mc.balance(A)
        out[f"prim/balance/{n}/A"] = A
        out[f"prim/balance/{n}/B"] = B
        out[f"prim/balance/{n}/scale"] = T.scale
        out[f"prim/onenorm/{n}/val"] = np.array(mc.onenorm(A))
    # estimator
    for n in (1, 2, 3, 9, 32, 64):
        for p in (1, 2, 7, 14):
            M = rng.standard_normal((n, n)) / np.sqrt(n)
            c = mc.OpCounter()
            v = mc.est_power_norm(M, p, counter=c)
            key = f"prim/est_power/{n}/{p}"
            out[key + "/M"] = M
            out[key + "/val"] = np.array(v)
            out[key + "/passes"] = np.array(c.estimation_passes)
        M1 = rng.standard_normal((n, n)) / np.sqrt(n)
        M2 = rng.standard_normal((n, n)) / np.sqrt(n)
        c = mc.OpCounter()
        v = mc.est_product_norm([(M1, 7), (M2, 1)], counter=c)
        key = f"prim/est_product/{n}"
        out[key + "/M1"], out[key + "/M2"] = M1, M2
        out[key + "/val"] = np.array(v)
        out[key + "/passes"] = np.array(c.estimation_passes)
    # sqrt_db
    for n in (1, 2, 8, 32, 64):
        G = rng.standard_normal((n, n))
        A = np.eye(n) + 0.5 * G / max(1.0, np.linalg.norm(G, 2))
        c = mc.OpCounter()
        X = sq.sqrt_db(A, counter=c)
        out[f"prim/sqrt_db/{n}/A"] = A
        out[f"prim/sqrt_db/{n}/X"] = X
        out[f"prim/sqrt_db/{n}/divisions"] = np.array(c.divisions)
    # eval_degopt, shipped schemes k = 1..5, with and without first-product reuse
    for k in range(1, 6):
        for n in (3, 32):
            G = rng.standard_normal((n, n))
            X = 0.2 * G / np.linalg.norm(G, 2)
            s = sc.builtin_scheme(k)
            c = mc.OpCounter()
            Z = sc.eval_degopt(s, X, counter=c)
            c2 = mc.OpCounter()
            Z2 = sc.eval_degopt(s, X, counter=c2, first_product=X @ X)
            key = f"prim/degopt/{k}/{n}"
            out[key + "/X"] = X
            out[key + "/Z"] = Z
            out[key + "/Zfp"] = Z2
            out[key + "/products"] = np.array([c.products, c2.products])
    return out


def main():
    mc, sc, sq = load_reference()
    from oracle import driver as D
    out = prim_cases(mc, sc, sq)
    prims = RefPrims(mc, sc, sq)
    names = []
    fields = ("status", "s", "k", "db_iters", "products", "divisions", "estimation_passes",
              "norm_estimations")
    for name, A in driver_cases():
        L, rep = D.logm_status(A, prims)
        names.append(name)
        out[f"drv/{name}/A"] = A
        out[f"drv/{name}/L"] = L if L is not None else np.zeros((0, 0))
        out[f"drv/{name}/ints"] = np.array([rep[f] for f in fields], dtype=np.int64)
        out[f"drv/{name}/alpha_used"] = np.array(rep["alpha_used"])
        print(f"{name:16s} n={A.shape[0]:3d} " + " ".join(f"{f}={rep[f]}" for f in fields))
    out["drv_names"] = np.array(names)
    out["drv_fields"] = np.array(fields)
    path = os.path.join(HERE, "golden_v1.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
