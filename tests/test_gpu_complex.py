"""complex128 input (as_square, matcore.py:60-61): the GPU path runs the real 2n x 2n
embedding E(Z) = [[X, -Y], [Y, X]] through the same kernels with every decision taken on Z
(complex 1-norms, complex estimator signs, |z| balancing, the DB stop test on Z) and reads
log Z back from the blocks of log E(Z).  L and the reports (status, s, k, DB iterations and
counters, tests/parity.classify) are compared with the oracle's complex run (its complex
branch is pinned bit-for-bit to the reference primitives by
tests/golden/golden_complex_v1.npz)."""
import os

import numpy as np
import pytest

from tests.parity import classify, rel_err, tolerance

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2401_10089_b200 as lp  # noqa: E402
from oracle import driver as D  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden_complex_v1.npz")


def test_complex_golden_cases_vs_reference_composition():
    g = np.load(GOLD)
    for name in (str(s) for s in g["drv_names"]):
        A = g[f"drv/{name}/A"]
        ints = dict(zip((str(f) for f in g["drv_fields"]), g[f"drv/{name}/ints"]))
        L, reps = lp.logm_batched(A[None], lp.LogmOptions(raise_on_error=False))
        assert int(reps[0]["status"]) == int(ints["status"]), name
        _, rr = D.logm_status(A, D.default_prims())
        cls, gf, of = classify(reps[0], rr)
        assert cls in ("match", "exempt", "db_plateau"), (name, cls, gf, of)
        if ints["status"] == 0:
            Lref = g[f"drv/{name}/L"]
            assert L.dtype == np.complex128
            assert rel_err(L[0], Lref) <= tolerance(A, Lref), (name, rel_err(L[0], Lref))
        else:
            assert np.isnan(L[0].real).all()


@pytest.mark.parametrize("n,B", [(8, 16), (33, 8), (100, 4)])
def test_complex_batches_vs_oracle_and_torch_io(n, B):
    rng = np.random.default_rng(n)
    G = (rng.standard_normal((B, n, n)) + 1j * rng.standard_normal((B, n, n))) / np.sqrt(2 * n)
    A = np.eye(n)[None] + 0.8 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    L, reps = lp.logm_batched(A)
    Lt, rt = lp.logm_batched(torch.from_numpy(A).cuda())          # torch complex in, out
    assert Lt.is_cuda and Lt.dtype == torch.complex128
    assert np.array_equal(Lt.cpu().numpy(), L) and rt.tobytes() == reps.tobytes()
    classes = []
    for b in range(B):
        Lr, rr = D.logm_status(A[b], D.default_prims())
        assert rr["status"] == 0 and int(reps[b]["status"]) == 0
        cls, g, o = classify(reps[b], rr)
        assert cls in ("match", "exempt", "db_plateau"), (b, cls, g, o)
        classes.append(cls)
        assert rel_err(L[b], Lr) <= tolerance(A[b], Lr), (b, rel_err(L[b], Lr))
    assert classes.count("match") >= B - 1, classes  # the decisions are Z's, not E(Z)'s
    L1, r1 = lp.logm(A[0])                                          # single-matrix entry point
    assert np.array_equal(L1, L[0]) and r1.s == int(reps[0]["s"])


@pytest.mark.parametrize("n,B", [(48, 6), (160, 2), (256, 2)])
def test_complex_nonnormal_reports_vs_oracle(n, B):
    """Complex A = S T S^-1 (T upper triangular with a log-uniform complex spectrum): several
    square roots and scaling-loop estimates, through G1 (embedding n <= 256 ... 320) and G2
    (embedding 512); the reports must match the oracle's complex run record by record."""
    rng = np.random.default_rng(1000 + n)
    As = []
    for _ in range(B):
        mag = np.exp(rng.uniform(np.log(1e-2), np.log(1e2), n))
        ph = rng.uniform(-2.5, 2.5, n)
        T = np.diag(mag * np.exp(1j * ph)) + np.triu((0.3 / n) * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))), 1)
        S = np.eye(n) + 0.1 * (rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))) / np.sqrt(n)
        As.append(S @ T @ np.linalg.inv(S))
    A = np.stack(As)
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    for b in range(B):
        Lr, rr = D.logm_status(A[b], D.default_prims())
        assert rr["status"] == 0, rr
        cls, g, o = classify(reps[b], rr)
        assert cls in ("match", "exempt", "db_plateau"), (b, cls, g, o)
        assert g["s"] >= 2, g
        assert rel_err(L[b], Lr) <= tolerance(A[b], Lr), (b, rel_err(L[b], Lr))
