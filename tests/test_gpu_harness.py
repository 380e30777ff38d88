"""Harness / CLI on the GPU (SPEC.md:515-562 examples): logm command, bench records, Er."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import cli, constants as C, harness, matio  # noqa: E402


def test_cmd_logm_identity_known_log_and_singular(tmp_path, capsys):
    p = tmp_path / "I.txt"
    matio.write_matrix(str(p), np.eye(6))
    out = tmp_path / "L.txt"
    assert cli.main(["logm", str(p), "-o", str(out)]) == 0
    assert np.array_equal(matio.read_matrix(str(out)), np.zeros((6, 6)))
    err = capsys.readouterr().err
    assert "s: 0" in err and "k: 1" in err
    A, L = harness.gen_test_matrices("b", 11, 24)
    matio.write_matrix(str(tmp_path / "A.txt"), A[0])
    matio.write_matrix(str(tmp_path / "Lref.txt"), L[0])
    assert cli.main(["logm", str(tmp_path / "A.txt"), "-o", str(out), "--ref", str(tmp_path / "Lref.txt")]) == 0
    er = float([ln for ln in capsys.readouterr().err.splitlines() if ln.startswith("Er:")][0].split()[1])
    assert er <= 1e-12
    Z = np.eye(4)
    Z[2, :] = 0.0
    matio.write_matrix(str(tmp_path / "Z.txt"), Z)
    assert cli.main(["logm", str(tmp_path / "Z.txt")]) == 3
    assert "singular" in capsys.readouterr().err


def test_cmd_bench_family_b_records(tmp_path):
    """bench on family (b), n = 32, 20 matrices -> all Er <= 1e-10."""
    out = tmp_path / "recs.csv"
    assert cli.main(["bench", "--family", "b", "--n", "32", "--count", "20", "--seed", "1", "-o", str(out)]) == 0
    recs = harness.records_from_csv(out.read_text())
    assert len(recs) == 20 and all(r.status == 0 and r.er <= 1e-10 for r in recs)
    assert all(r.equivalent_m == r.products + 4.0 * r.divisions / 3.0 for r in recs)
    # performance profile over two copies of the same method set: p = 1 everywhere
    prof = harness.performance_profile({r.matrix_id: {"gpu": r.er, "gpu2": r.er} for r in recs})
    assert all(p == 1.0 for pts in prof.values() for _, p in pts)


def test_family_c_bidiagonal_and_selection_invariant():
    """family (c), superdiagonal 5, n = 8: logm succeeds, alpha <= Theta_k;
    SPEC.md:594 (#7): when s >= 1 the evaluation uses exactly k - 1 products."""
    A, _ = harness.gen_test_matrices("c", 0, 8, superdiag=5.0)
    L, reps = lp.logm_batched(A)
    r = reps[0]
    assert r["status"] == 0 and r["alpha_used"] <= C.THETA[r["k"] - 1]
    if r["s"] >= 1:
        assert r["products"] == r["k"] - 1
    E = torch.linalg.matrix_exp(torch.from_numpy(np.asarray(L)[0]).cuda()).cpu().numpy()
    assert np.linalg.norm(E - A[0]) <= 1e-12 * np.linalg.norm(A[0])


@pytest.mark.parametrize("n", [32, 96])
def test_relative_error_batched_matches_host(n):
    A, L = harness.gen_test_matrices("b", 5, n, count=4)
    Lg, _ = lp.logm_batched(A)
    Lg = np.asarray(Lg)
    dev = harness.relative_error_batched(torch.from_numpy(Lg).cuda(), torch.from_numpy(L).cuda())
    host = np.array([harness.relative_error(Lg[q], L[q]) for q in range(4)])
    assert np.allclose(dev, host, rtol=1e-6, atol=0) and (host <= 1e-11).all()


def test_expm_ref_batched_and_round_trip():
    """SPEC.md:592 (#5): n = 128, ||A|| = 0.5: ||expm_ref(logm(I + A)) - (I + A)|| <= 1e-13."""
    from paper_2401_10089_b200.validate import expm_ref_batched
    A, _ = harness.gen_test_matrices("a", 3, 128, count=3)
    Ad = torch.from_numpy(A).cuda()
    L, reps = lp.logm_batched(Ad)
    E = expm_ref_batched(L)
    res = torch.linalg.matrix_norm(E - Ad, ord=2) / torch.linalg.matrix_norm(Ad, ord=2)
    assert (reps["status"] == 0).all() and float(res.max()) <= 1e-13
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((4, 20, 20)) * 3.0).cuda()
    ref = torch.linalg.matrix_exp(X)
    got = expm_ref_batched(X)
    assert float((torch.linalg.matrix_norm(got - ref) / torch.linalg.matrix_norm(ref)).max()) <= 1e-12


def test_spectrum_precheck(tmp_path, capsys):
    from paper_2401_10089_b200.validate import spectrum_violations
    rng = np.random.default_rng(2)
    from paper_2401_10089_b200 import synth
    S = synth.spd(rng, 10, -1, 1)
    N = np.diag([-1.0, 2.0, 3.0])
    Z = np.diag([0.0, 1.0, 2.0])
    assert list(spectrum_violations(np.stack([np.eye(3), N, Z]))) == [False, True, True]
    assert not spectrum_violations(torch.from_numpy(S).cuda())[0]
    with pytest.raises(lp.SpectrumError):
        lp.logm(N, lp.LogmOptions(check_spectrum=True))
    _, reps = lp.logm_batched(np.stack([np.eye(3), N]), lp.LogmOptions(check_spectrum=True, raise_on_error=False))
    assert list(reps["status"]) == [0, 5]
    matio.write_matrix(str(tmp_path / "N.txt"), N)
    assert cli.main(["logm", str(tmp_path / "N.txt"), "--check-spectrum"]) == 3
    assert "spectrum" in capsys.readouterr().err


def _expm_ref_np(A):
    """numpy restatement of the reference's expm_ref (matcore.py:318-336) -- test oracle."""
    import math
    nrm = np.abs(A).sum(axis=0).max()
    s = 0 if nrm <= 0.5 else max(0, int(math.ceil(math.log2(nrm / 0.5))))
    X = A / (2.0 ** s)
    E = np.eye(A.shape[0])
    T = E.copy()
    for j in range(20, 0, -1):
        T = E + (X @ T) / j
    for _ in range(s):
        T = T @ T
    return T


@pytest.mark.parametrize("n,scale", [(20, 3.0), (71, 0.2), (130, 1.5), (64, 0.0)])
def test_expm_ref_kernels_vs_reference_recipe(n, scale):
    """lgm_expm_ref_f64 (the library's kernels) against the reference recipe in numpy: same
    scaling exponent per matrix (s from 0 to ~8 here), 1e-13 relative agreement."""
    from paper_2401_10089_b200.validate import expm_ref_batched
    rng = np.random.default_rng(n)
    X = rng.standard_normal((3, n, n)) * scale / np.sqrt(n)
    X[1] *= 10.0
    got = expm_ref_batched(torch.from_numpy(X).cuda()).cpu().numpy()
    for b in range(3):
        ref = _expm_ref_np(X[b])
        assert np.linalg.norm(got[b] - ref) / np.linalg.norm(ref) <= 1e-13, b


def test_spectrum_check_kernel_vs_numpy_eigvals():
    """lgm_spectrum_check_f64 (Hessenberg + Francis QR on the device) against numpy's eigvals
    (LAPACK dgeev, what eig_small calls) on matrices with clear-cut spectra."""
    from paper_2401_10089_b200.validate import spectrum_check
    rng = np.random.default_rng(3)
    mats, want = [], []
    for n in (1, 2, 5, 17, 64, 100, 257):
        for kind in range(4):
            Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
            lam = rng.uniform(0.5, 3.0, n)
            if kind == 1:
                lam[rng.integers(n)] = -rng.uniform(0.5, 2.0)        # one negative real eigenvalue
            A = (Q * lam) @ Q.T
            if kind == 2 and n >= 2:                                    # complex pairs, positive reals
                R = np.eye(n)
                R[:2, :2] = [[1.0, -2.0], [2.0, 1.0]]
                A = Q @ R @ np.diag(lam) @ Q.T
            if kind == 3:                                               # nonnormal, shifted spectrum
                A = rng.standard_normal((n, n)) / np.sqrt(n) + 3.0 * np.eye(n)
                if n >= 5:
                    A[0, 0] = -10.0
            ev = np.linalg.eigvals(A)
            mats.append(A)
            want.append(bool(((ev.imag == 0) & (ev.real <= 0)).any()))
    for A, w in zip(mats, want):
        assert spectrum_check(A)[0] == int(w), (A.shape, w)
    batch = np.stack([m for m in mats if m.shape[0] == 17])
    assert list(spectrum_check(batch)) == [int(w) for m, w in zip(mats, want) if m.shape[0] == 17]
