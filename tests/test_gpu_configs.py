"""GPU-vs-oracle parity on the BASELINE.json configurations as written.

Every test runs the CUDA path through ``logm_batched`` (C ABI) and the CPU oracle
(oracle/driver.py over oracle/primitives.py, pinned to the reference's own primitives by
tests/golden) on the same seeded inputs, then applies tests/parity.py: status, s, k,
db_iters, products, divisions, estimation_passes and norm_estimations equal per matrix
(margin exemption < 1e-10 only; db_plateau only for iteration-count noise with equal
status / s / k), and ||L_gpu - L_ref||_F / ||L_ref||_F <= max(1e-12, 10 cond_log u).

The oracle runs on all host cores (process pool); the n = 4096 cases run one matrix with
all-core BLAS (about a minute each on the GPU box's host).
"""
import numpy as np
import pytest

from tests.parity import check_batch

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402

NOFAIL = lp.LogmOptions(raise_on_error=False)


def _run(A):
    return lp.logm_batched(torch.from_numpy(A).cuda(), NOFAIL)


def _host(L):
    return L.cpu().numpy()


def test_config2_full_batch_vs_oracle():
    """Config 2 as written: all 4096 near-identity 32 x 32 matrices (Engine F)."""
    A = synth.config(2)
    L, reps = _run(A)
    counts, _ = check_batch(A, _host(L), reps)
    assert counts["match"] + counts["db_plateau"] + counts["exempt"] == 4096


def test_config1_as_written_vs_oracle():
    A = synth.config(1)
    L, reps = _run(A)
    counts, _ = check_batch(A, _host(L), reps)
    assert counts["match"] == 1


def test_config3_as_written_status_parity():
    """Config 3 as written (n = 128, kappa ~ 1e18): the reference's sqrt_db does not converge
    (SURVEY.md 8(d)); status DB_NOCONV after 50 iterations on both sides, same s, same
    estimator work before the failing root."""
    A = synth.config(3, batch=16)
    L, reps = _run(A)
    counts, res = check_batch(A, _host(L), reps)
    assert counts["mismatch"] == 0
    for b, (rr, _, _) in enumerate(res):
        assert rr["status"] == 2 and int(reps[b]["status"]) == 2
        assert int(reps[b]["db_iters"]) == rr["db_iters"]
        assert np.isnan(_host(L)[b]).all()          # failed entries are NaN, never stale data


def test_config3b_vs_oracle():
    A = synth.config("3b", batch=32)
    L, reps = _run(A)
    counts, _ = check_batch(A, _host(L), reps)
    assert counts["match"] + counts["db_plateau"] >= 30


def test_config4_16_matrices_vs_oracle():
    """Config 4 (n = 512 SPD, lambda in [1e-4, 1e4]): the first 16 of its 256 matrices."""
    A = synth.config(4, batch=16)
    L, reps = _run(A)
    counts, _ = check_batch(A, _host(L), reps)
    assert counts["mismatch"] == 0


def test_config5b_one_matrix_vs_oracle():
    """Config 5b (n = 4096, well-conditioned S T S^-1), one matrix: exercises the G2
    cluster-panel inversion, the rank-64 passes and the n > 512 estimator end to end."""
    A = synth.config("5b", batch=1)
    L, reps = _run(A)
    counts, _ = check_batch(A, _host(L), reps)
    assert counts["mismatch"] == 0 and int(reps[0]["status"]) == 0


def test_config5_as_written_status_parity():
    """Config 5 as written (n = 4096, kappa ~ 1e23): DB_NOCONV with 50 iterations on both
    sides (the reference raised ConvergenceError after 50 DB iterations)."""
    A = synth.config(5, batch=1)
    L, reps = _run(A)
    counts, res = check_batch(A, _host(L), reps)
    rr = res[0][0]
    assert counts["mismatch"] == 0
    assert rr["status"] == 2 and int(reps[0]["status"]) == 2
    assert int(reps[0]["db_iters"]) == rr["db_iters"]
    assert int(reps[0]["s"]) == rr["s"]
