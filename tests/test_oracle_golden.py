"""Pin the oracle (oracle/) to the reference: golden fixtures + SPEC known answers.

CPU only.  The fixtures in tests/golden/golden_v1.npz were produced by the
reference's own primitives (tests/golden/make_golden.py); the restated primitives
must reproduce them (same numpy/scipy call sequence => same bits on this image; a
1e-13 relative tolerance is allowed for the BLAS/LAPACK-dependent ones in case the
suite runs on a host whose OpenBLAS picks a different kernel).
"""
import math
import os

import numpy as np
import pytest

from oracle import driver as D
from oracle import primitives as P
from paper_2401_10089_b200 import constants as C

U = 2.0 ** -53


def _close(a, b, rtol=1e-13):
    a = np.asarray(a)
    b = np.asarray(b)
    assert a.shape == b.shape
    if np.array_equal(a, b):
        return
    scale = max(np.abs(b).max(), 1e-300)
    assert np.abs(a - b).max() <= rtol * scale


# ----------------------------------------------------------------- primitives vs reference

@pytest.mark.parametrize("n", [1, 5, 17, 32, 64, 130])
def test_balance_matches_reference_bitwise(golden, n):
    A = golden[f"prim/balance/{n}/A"]
    B, scale, _ = P.balance(A)
    assert np.array_equal(B, golden[f"prim/balance/{n}/B"])
    assert np.array_equal(scale, golden[f"prim/balance/{n}/scale"])
    assert P.onenorm(A) == float(golden[f"prim/onenorm/{n}/val"])


@pytest.mark.parametrize("n", [1, 2, 3, 9, 32, 64])
@pytest.mark.parametrize("p", [1, 2, 7, 14])
def test_est_power_norm_matches_reference(golden, n, p):
    key = f"prim/est_power/{n}/{p}"
    c = P.Counter()
    v = P.est_power_norm(golden[key + "/M"], p, counter=c)
    _close(v, golden[key + "/val"])
    assert c.estimation_passes == int(golden[key + "/passes"])


@pytest.mark.parametrize("n", [1, 2, 3, 9, 32, 64])
def test_est_product_norm_matches_reference(golden, n):
    key = f"prim/est_product/{n}"
    c = P.Counter()
    v = P.est_product_norm([(golden[key + "/M1"], 7), (golden[key + "/M2"], 1)], counter=c)
    _close(v, golden[key + "/val"])
    assert c.estimation_passes == int(golden[key + "/passes"])


@pytest.mark.parametrize("n", [1, 2, 8, 32, 64])
def test_sqrt_db_matches_reference(golden, n):
    c = P.Counter()
    X, its = P.sqrt_db(golden[f"prim/sqrt_db/{n}/A"], counter=c)
    _close(X, golden[f"prim/sqrt_db/{n}/X"])
    assert c.divisions == int(golden[f"prim/sqrt_db/{n}/divisions"]) == 2 * its


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
@pytest.mark.parametrize("n", [3, 32])
def test_eval_degopt_matches_reference(golden, k, n):
    key = f"prim/degopt/{k}/{n}"
    X = golden[key + "/X"]
    c1, c2 = P.Counter(), P.Counter()
    Z = P.eval_degopt(C.SCHEMES[k - 1], X, counter=c1)
    Z2 = P.eval_degopt(C.SCHEMES[k - 1], X, counter=c2, first_product=X @ X)
    _close(Z, golden[key + "/Z"])
    _close(Z2, golden[key + "/Zfp"])
    assert [c1.products, c2.products] == list(golden[key + "/products"])


# ----------------------------------------------------------------- driver vs reference-composed driver

def _drv_names(golden):
    return [str(s) for s in golden["drv_names"]]


def test_driver_matches_reference_composed(golden):
    fields = [str(f) for f in golden["drv_fields"]]
    for name in _drv_names(golden):
        A = golden[f"drv/{name}/A"]
        L, rep = D.logm_status(A, D.default_prims())
        ints = [rep[f] for f in fields]
        assert ints == list(golden[f"drv/{name}/ints"]), name
        if rep["status"] == 0:
            _close(L, golden[f"drv/{name}/L"])
            assert rep["alpha_used"] == pytest.approx(float(golden[f"drv/{name}/alpha_used"]),
                                                      rel=1e-12, abs=0)


# ----------------------------------------------------------------- SPEC known answers

def test_theta_frozen_from_shipped_coefficients():
    # theta_for_scheme at 300 digits on the shipped files; Table 2 within 2%
    table2 = (1.83e-8, 1.53e-4, 1.33e-2, 9.31e-2, 0.246)
    for t, p in zip(C.THETA, table2):
        assert abs(t - p) / p < 0.02
    assert C.ORDER[:5] == (2, 4, 8, 14, 14) and C.K_DEFAULT == 5
    # k = 6..9 (generated, opt-in): Theta grows with k and every order is even (Algorithm 1's
    # alpha / max_in formulas)
    assert all(a < b for a, b in zip(C.THETA, C.THETA[1:])) and all(m % 2 == 0 for m in C.ORDER)


def test_spec_onenorm_and_det():
    assert P.onenorm(np.array([[1.0, -2.0], [3.0, 4.0]])) == 6.0
    fac, lad = P.lu_logabsdet(np.diag([2.0, 3.0]))
    assert math.exp(lad) == pytest.approx(6.0, rel=1e-15)


def test_spec_est_power_norm_examples():
    D4 = np.diag([0.5, -2.0, 1.5, 0.1])
    assert P.est_power_norm(D4, 3) == pytest.approx(8.0, rel=1e-15)
    assert P.est_power_norm(np.zeros((4, 4)), 5) == 0.0
    rng = np.random.default_rng(3)
    for _ in range(200):
        M = rng.standard_normal((8, 8))
        true = np.abs(np.linalg.matrix_power(M, 4)).sum(axis=0).max()
        est = P.est_power_norm(M, 4)
        assert true / 10.0 <= est <= true * (1 + 1e-12)


def test_spec_sqrt_db_examples():
    X, its = P.sqrt_db(np.eye(6))
    assert its == 1 and np.array_equal(X, np.eye(6))
    X, _ = P.sqrt_db(np.diag([4.0, 9.0]))
    assert np.abs(X - np.diag([2.0, 3.0])).max() <= 100 * U * 3


def test_spec_eval_degopt_examples():
    k5 = C.SCHEMES[4]
    c = P.Counter()
    z = P.eval_degopt(k5, np.array([[0.2]]), counter=c)
    assert abs(z[0, 0] + math.log(0.8)) <= 10 * U * abs(math.log(0.8))
    assert c.products == 5
    assert np.array_equal(P.eval_degopt(k5, np.zeros((3, 3))), np.zeros((3, 3)))
    x = 0.1
    z2 = P.eval_degopt(C.SCHEMES[1], np.array([[x]]))
    assert z2[0, 0] == pytest.approx(x + x**2 / 2 + x**3 / 3 + x**4 / 4, rel=1e-15)


def test_spec_balance_examples():
    S = np.array([[2.0, 1.0, 0.5], [1.0, 3.0, 0.2], [0.5, 0.2, 1.0]])
    B, scale, _ = P.balance(S)
    assert np.array_equal(scale, np.ones(3)) and np.array_equal(B, S)
    rng = np.random.default_rng(5)
    d = 2.0 ** rng.integers(-10, 10, 6)
    A = rng.standard_normal((6, 6)) * (d[:, None] / d[None, :])
    B, scale, _ = P.balance(A)
    assert np.array_equal(P.unbalance(B, scale), A)


def test_spec_logm_identity():
    L, rep = D.logm(np.eye(4))
    assert np.array_equal(L, np.zeros((4, 4)))
    assert (rep["s"], rep["k"], rep["alpha_used"]) == (0, 1, 0.0)


def test_spec_logm_known_log_and_invariants():
    from paper_2401_10089_b200 import synth
    rng = np.random.default_rng(11)
    for n in (16, 24, 40):                                                   # SPEC.md:453, acceptance 6
        A, Lex = synth.known_log(rng, n, kappa=10.0)
        L, rep = D.logm(A)
        er = np.linalg.norm(L - Lex, 2) / np.linalg.norm(Lex, 2)
        assert er <= 1e3 * 10.0 ** 2 * U
        # acceptance 7: alpha_used <= Theta_k, product accounting
        assert rep["alpha_used"] <= C.THETA[rep["k"] - 1]
        assert rep["products"] == (rep["k"] - 1 if rep["s"] >= 1 else rep["k"])


def test_spec_logm_roundtrip_n128():
    # SPEC.md:454 / acceptance 5: ||expm(logm(I+A)) - (I+A)|| <= 1e-13 with ||A|| = 0.5
    import scipy.linalg
    rng = np.random.default_rng(12)
    G = rng.standard_normal((128, 128))
    A = np.eye(128) + 0.5 * G / np.linalg.norm(G, 2)
    L, rep = D.logm(A)
    assert np.linalg.norm(scipy.linalg.expm(L) - A, 2) <= 1e-13


def test_logm_failure_statuses(golden):
    L, rep = D.logm_status(np.array([[1.0, np.nan], [0.0, 1.0]]), D.default_prims())
    assert rep["status"] == D.NONFINITE and L is None
    with pytest.raises(ValueError):
        D.logm(np.ones((2, 3)))
    with pytest.raises(P.ConvergenceError):
        D.logm(np.diag([-1.0, 2.0]))


def test_oracle_complex_branch_vs_reference_primitives():
    """complex128 (matcore.py:60-61, complex sign matcore.py:226-231): the restated driver over
    the restated primitives reproduces the restated driver over the reference's own primitives
    (tests/golden/golden_complex_v1.npz, make_golden_complex.py) bit for bit."""
    from oracle import driver as D
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_complex_v1.npz"))
    fields = [str(f) for f in g["drv_fields"]]
    for name in (str(s) for s in g["drv_names"]):
        A = g[f"drv/{name}/A"]
        L, rep = D.logm_status(A, D.default_prims())
        assert [rep[f] for f in fields] == list(g[f"drv/{name}/ints"]), name
        if rep["status"] == 0:
            assert L.dtype == np.complex128 and np.array_equal(L, g[f"drv/{name}/L"]), name
    M = g["prim/est/M"]
    for p in (1, 3, 8):
        c = P.Counter()
        v = P.est_power_norm(M, p, counter=c)
        assert [v, c.estimation_passes] == list(g[f"prim/est/{p}"])
    X, _ = P.sqrt_db(g["prim/sqrt/A"])
    assert np.array_equal(X, g["prim/sqrt/X"])
    B, sc, _ = P.balance(g["prim/bal/A"])
    assert np.array_equal(B, g["prim/bal/B"]) and np.array_equal(sc, g["prim/bal/scale"])
