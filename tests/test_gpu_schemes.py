"""Schemes k = 6..K_MAX (generated with the reference's fit_minmax + moment matching,
tools/gen_schemes.py; opt-in through LogmOptions.max_k): GPU vs the oracle on the same
coefficient bits.  Parity for k > 5 is pinned by the oracle restatement only (the reference
ships no such schemes), so these are consistency tests of the two implementations plus the
accuracy bar against the oracle's logarithm."""
import numpy as np
import pytest

from tests.parity import check_batch, rel_err

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2401_10089_b200 as lp  # noqa: E402
from oracle import primitives as P  # noqa: E402
from paper_2401_10089_b200 import constants as C  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402

KS = list(range(C.K_DEFAULT + 1, C.K_MAX + 1))
if not KS:  # pragma: no cover
    pytest.skip("no schemes beyond k = 5 generated", allow_module_level=True)


@pytest.mark.parametrize("n", [24, 64, 100])
@pytest.mark.parametrize("k", KS)
def test_eval_degopt_high_k(n, k):
    rng = np.random.default_rng(10 * n + k)
    G = rng.standard_normal((2, n, n))
    X = 0.3 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    c = lp.OpCounter()
    Z = lp.eval_degopt(k, X, counter=c)
    c2 = lp.OpCounter()
    Z2 = lp.eval_degopt(k, X, counter=c2, first_product=X @ X)
    for b in range(2):
        Zo = P.eval_degopt(C.SCHEMES[k - 1], X[b])
        assert rel_err(Z[b], Zo) <= 1e-13 and rel_err(Z2[b], Zo) <= 1e-13
    assert c.products == 2 * k and c2.products == 2 * (k - 1)


@pytest.mark.parametrize("c,n,B", [(2, 32, 128), ("3b", 48, 16), ("3b", 128, 16), (4, 512, 4), (1, 64, 1)])
def test_logm_max_k_high_vs_oracle(c, n, B):
    A = synth.config(c, batch=B, n=n)
    opts = lp.LogmOptions(max_k=C.K_MAX, raise_on_error=False)
    L, reps = lp.logm_batched(A, opts)
    counts, _ = check_batch(A, L, reps, max_k=C.K_MAX)
    assert counts["mismatch"] == 0
    # the wider Theta buys square roots: never more than with the shipped k <= 5
    _, reps5 = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    ok = (reps["status"] == 0) & (reps5["status"] == 0)
    assert (reps["s"][ok] <= reps5["s"][ok]).all()
    assert (reps["alpha_used"][ok] <= np.array(C.THETA)[reps["k"][ok] - 1]).all()


@pytest.mark.parametrize("n", [24, 64, 100])
@pytest.mark.parametrize("k", [1, 3, 5, 7])
def test_eval_degopt_caller_scheme(n, k):
    """Any GraphScheme (schemes.py:50-126) through lgm_eval_degopt_scheme_f64: random
    coefficients (first rows pinned to (0, 1) so first_product applies), GPU vs the oracle's
    eval_degopt on the same coefficients; an unnormalized scheme with first_product raises."""
    rng = np.random.default_rng(100 * n + k)
    rows = lambda: tuple([(0.0, 1.0)] + [tuple(0.5 * rng.standard_normal(j + 2)) for j in range(1, k)])  # noqa: E731
    s = lp.GraphScheme(lhs=rows(), rhs=rows(), out=tuple(0.5 * rng.standard_normal(k + 2)))
    G = rng.standard_normal((2, n, n))
    X = 0.3 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    c, c2 = lp.OpCounter(), lp.OpCounter()
    Z = lp.eval_degopt(s, X, counter=c)
    Z2 = lp.eval_degopt(s, X, counter=c2, first_product=X @ X)
    for b in range(2):
        Zo = P.eval_degopt((s.lhs, s.rhs, s.out), X[b])
        assert rel_err(Z[b], Zo) <= 1e-13 and rel_err(Z2[b], Zo) <= 1e-13, (rel_err(Z[b], Zo), rel_err(Z2[b], Zo))
    assert c.products == 2 * k and c2.products == 2 * (k - 1)
    # the built-in path is untouched by a caller's scheme call (its coefficients live in the call)
    Zb = lp.eval_degopt(k, X)
    for b in range(2):
        assert rel_err(Zb[b], P.eval_degopt(C.SCHEMES[k - 1], X[b])) <= 1e-13
    bad = lp.GraphScheme(lhs=((0.5, 1.0),) + s.lhs[1:], rhs=s.rhs, out=s.out)
    with pytest.raises(ValueError):
        lp.eval_degopt(bad, X, first_product=X @ X)
