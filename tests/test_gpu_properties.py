"""Property-based GPU tests (hypothesis, derandomized) of the SPEC's invariants for the hot path:
SPEC.md:112-116 (estimator on diagonals, balance round trip), :196-198 (eval_degopt product
count, 1x1 scalar agreement), :239-242 (sqrt_db residual, mu = 1 on I, commutation) and
:483-487 (alpha_used <= Theta_k, product accounting, radix-diagonal scaling invariance,
logm(A^2) = 2 logm(A)).  Sizes straddle both engines (Engine F n <= 64, Engine G n > 64)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from hypothesis import given, settings, strategies as st  # noqa: E402

import paper_2401_10089_b200 as lp  # noqa: E402
from oracle import primitives as P  # noqa: E402
from paper_2401_10089_b200 import constants as C  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402

U = 2.0 ** -53
FAST = settings(max_examples=20, deadline=None, derandomize=True)
sizes = st.sampled_from([1, 2, 5, 16, 31, 32, 33, 64, 65, 96])
seeds = st.integers(min_value=0, max_value=2 ** 31 - 1)


@FAST
@given(n=sizes, seed=seeds, p=st.integers(min_value=1, max_value=15))
def test_est_power_norm_exact_on_diagonals(n, seed, p):
    d = np.random.default_rng(seed).uniform(-2.0, 2.0, n)
    e = lp.est_power_norm(np.diag(d), p)
    assert e == pytest.approx(float(np.max(np.abs(d)) ** p), rel=1e-13)


@FAST
@given(n=sizes, seed=seeds)
def test_balance_round_trip_exact(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n)) * (10.0 ** rng.uniform(-3, 3, n))[None, :]
    B, T = lp.balance(A)
    assert np.array_equal(T.revert(B), A)                       # radix-2 scales: exact


@FAST
@given(k=st.integers(min_value=1, max_value=C.K_MAX), x=st.floats(min_value=-0.3, max_value=0.3))
def test_eval_degopt_products_and_scalar(k, x):
    ctr = lp.OpCounter()
    Z = lp.eval_degopt(k, np.array([[x]]), counter=ctr)
    assert ctr.products == k
    ref = float(np.asarray(P.eval_degopt(C.SCHEMES[k - 1], np.array([[x]]))).reshape(-1)[0])
    got = float(np.asarray(Z).reshape(-1)[0])
    assert abs(got - ref) <= 4 * U * max(abs(ref), U)


@FAST
@given(n=sizes, seed=seeds)
def test_sqrt_db_residual_and_commutation(n, seed):
    rng = np.random.default_rng(seed)
    G = rng.standard_normal((n, n))
    A = np.eye(n) + 0.4 * G / max(np.linalg.norm(G, 2), 1e-300)
    X = lp.sqrt_db(A)
    na, nx = np.linalg.norm(A, 1), np.linalg.norm(X, 1)
    kappa = na * np.linalg.norm(np.linalg.inv(A), 1)
    assert np.linalg.norm(X @ X - A, 1) / na <= max(10 * n * U, 1e3 * U * kappa)
    assert np.linalg.norm(X @ A - A @ X, 1) <= 1e3 * U * na * nx


@pytest.mark.parametrize("n", [1, 7, 32, 80])
def test_sqrt_db_identity_one_iteration(n):
    X, it, stt = lp.sqrt_db_batched(np.eye(n)[None])
    assert np.array_equal(X[0], np.eye(n)) and int(it[0]) == 1 and int(stt[0]) == 0


@FAST
@given(n=sizes, seed=seeds)
def test_logm_selection_invariants(n, seed):
    rng = np.random.default_rng(seed)
    A = np.stack([synth.near_identity(rng, n), synth.spd(rng, n, -1.5, 1.5)])
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    for r in reps:
        assert r["status"] == 0
        assert r["alpha_used"] <= C.THETA[r["k"] - 1]
        assert r["products"] == (r["k"] - 1 if r["s"] >= 1 else r["k"])


@FAST
@given(n=sizes, seed=seeds)
def test_logm_radix_scaling_invariance_on_diagonals(n, seed):
    """Diagonal A: logm(D A D^-1) = logm(A) selects the same (s, k), balancing off."""
    rng = np.random.default_rng(seed)
    d = 10.0 ** rng.uniform(-1.0, 1.0, n)
    D = np.diag(2.0 ** rng.integers(-8, 9, n).astype(np.float64))
    A = np.diag(d)
    opts = lp.LogmOptions(balance=False, raise_on_error=False)
    _, r1 = lp.logm_batched(A[None], opts)
    _, r2 = lp.logm_batched((D @ A @ np.linalg.inv(D))[None], opts)
    assert (int(r1[0]["s"]), int(r1[0]["k"])) == (int(r2[0]["s"]), int(r2[0]["k"]))


@FAST
@given(n=st.sampled_from([4, 16, 33, 64, 72]), seed=seeds)
def test_logm_square_identity_spd(n, seed):
    S = synth.spd(np.random.default_rng(seed), n, -1.0, 1.0)
    L, _ = lp.logm_batched(np.stack([S, S @ S]))
    assert np.linalg.norm(L[1] - 2 * L[0]) / np.linalg.norm(2 * L[0]) <= 1e4 * U
