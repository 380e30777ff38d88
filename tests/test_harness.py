"""Harness / CLI host logic -- CPU only.

Matrix text I/O is pinned byte-for-byte to the reference's own serializer
(tests/golden/matio_ref*.txt, written by tests/golden/make_matio_golden.py through
logmpoly.matcore.format_matrix); the rest follows the SPEC's examples.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

from paper_2401_10089_b200 import cli, harness, matio  # noqa: E402
from paper_2401_10089_b200.exceptions import SchemeFormatError  # noqa: E402
from make_matio_golden import matrices  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")


def test_format_matrix_matches_reference_bytes():
    M, Z = matrices()
    assert matio.format_matrix(M) == open(os.path.join(GOLD, "matio_ref.txt")).read()
    assert matio.format_matrix(Z) == open(os.path.join(GOLD, "matio_ref_complex.txt")).read()


def test_parse_round_trip_bitwise():
    M, Z = matrices()
    R = matio.parse_matrix(open(os.path.join(GOLD, "matio_ref.txt")).read())
    assert R.dtype == np.float64 and np.array_equal(R.view(np.int64), M.view(np.int64))   # incl. -0.0
    C = matio.parse_matrix(open(os.path.join(GOLD, "matio_ref_complex.txt")).read())
    assert C.dtype == np.complex128 and np.array_equal(C, Z)
    text = "# comment\n\n2\n  1 2\n# mid\n3 4\n\n"
    assert np.array_equal(matio.parse_matrix(text), [[1.0, 2.0], [3.0, 4.0]])


@pytest.mark.parametrize("text", ["", "# only\n", "x\n1\n", "2\n1 2\n", "2\n1 2\n3\n", "1\nabc\n", "1\n1+i\n",
                                  "0\n"])
def test_parse_errors(text):
    with pytest.raises(SchemeFormatError):
        matio.parse_matrix(text)


def test_nonfinite_and_shape_rejected():
    with pytest.raises(ValueError):
        matio.format_matrix([[1.0, np.inf], [0.0, 1.0]])
    with pytest.raises(ValueError):
        matio.parse_matrix("1\nnan\n")
    with pytest.raises(ValueError):
        matio.format_matrix(np.ones((2, 3)))


def test_relative_error_examples():
    rng = np.random.default_rng(0)
    L = rng.standard_normal((32, 32))
    assert harness.relative_error(L, L) == 0.0
    assert abs(harness.relative_error(1.01 * L, L) - 0.01) <= 1e-12
    with pytest.raises(ValueError):
        harness.relative_error(L, np.zeros_like(L))


@pytest.mark.parametrize("n", [32, 65, 128])
def test_power_iteration_norm_vs_svd(n):
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n)) + np.diag(np.linspace(1, 3, n))
    s = np.linalg.svd(M, compute_uv=False)[0]
    assert abs(harness._power_norm2(M, steps=500, tol=1e-14) - s) <= 1e-8 * s
    # the SPEC's 50-step cap above n = 64 is a lower bound (close singular values converge slowly)
    est = harness.norm2(M)
    assert (abs(est - s) <= 1e-14 * s) if n <= 64 else (0.95 * s <= est <= s * (1 + 1e-14))


def test_performance_profile_examples():
    one = harness.performance_profile({"m0": {"A": 1e-15}, "m1": {"A": 2e-14}})
    assert all(p == 1.0 for _, p in one["A"])
    prof = harness.performance_profile({"m0": {"A": 1e-15, "B": 3e-15}})
    pA, pB = dict(prof["A"]), dict(prof["B"])
    assert pA[1.0] == 1.0
    assert all(pB[a] == 0.0 for a in pB if a < 3.0) and all(pB[a] == 1.0 for a in pB if a >= 3.0)
    low = harness.performance_profile({"m0": {"A": 1e-18, "B": 5e-17}})       # both floored to u
    assert dict(low["A"])[1.0] == 1.0 and dict(low["B"])[1.0] == 1.0
    for pts in prof.values():
        ps = [p for _, p in pts]
        assert ps == sorted(ps) and ps[-1] <= 1.0
    with pytest.raises(ValueError):
        harness.performance_profile({"m0": {"A": 1e-15, "B": 1e-15}, "m1": {"A": 1e-15}})


def test_gen_families_deterministic_and_known_log():
    import scipy.linalg
    for fam in "abcd":
        A1, L1 = harness.gen_test_matrices(fam, 7, 12, count=3)
        A2, L2 = harness.gen_test_matrices(fam, 7, 12, count=3)
        assert A1.shape == (3, 12, 12) and np.array_equal(A1, A2)
        assert (L1 is None) == (fam != "b")
    A, L = harness.gen_test_matrices("b", 3, 16, count=2)
    for q in range(2):
        E = scipy.linalg.expm(L[q])
        assert np.linalg.norm(E - A[q]) <= 1e-13 * np.linalg.norm(A[q])
    A, _ = harness.gen_test_matrices("a", 0, 20)
    assert abs(np.linalg.norm(A[0] - np.eye(20), 2) - 0.5) <= 1e-14
    A, _ = harness.gen_test_matrices("d", 0, 20)
    assert np.allclose(A[0], A[0].T, rtol=0, atol=0) and np.linalg.eigvalsh(A[0]).min() > 0


def test_records_csv_round_trip():
    recs = [harness.BenchRecord("m0", 32, "x", 1.0 / 3.0, 4, 22, 4 + 88 / 3, 1e-5, 0, 2, 5),
            harness.BenchRecord("m1", 32, "x", float("nan"), 0, 0, 0.0, 2e-5, 2, 0, 0)]
    back = harness.records_from_csv(harness.records_to_csv(recs))
    assert back[0] == recs[0]
    assert np.isnan(back[1].er) and back[1].status == 2


def test_cli_theta_gen_profile_and_input_errors(tmp_path, capsys):
    assert cli.main(["theta"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0] == "k,order_m,theta" and any(ln.startswith("5,14,0.2448") for ln in out)
    assert cli.main(["gen", "b", "--n", "6", "--count", "2", "--seed", "4", "--out-dir", str(tmp_path)]) == 0
    files = sorted(os.listdir(tmp_path))
    assert len(files) == 4 and any(f.endswith(".log.txt") for f in files)
    A = matio.read_matrix(str(tmp_path / files[0]))
    assert A.shape == (6, 6)
    csvp = tmp_path / "r.csv"
    csvp.write_text(harness.records_to_csv([harness.BenchRecord("m0", 4, "A", 1e-15, 0, 0, 0.0, 0.0),
                                             harness.BenchRecord("m0", 4, "B", 3e-15, 0, 0, 0.0, 0.0)]))
    assert cli.main(["profile", str(csvp)]) == 0
    prof = capsys.readouterr().out.splitlines()
    assert prof[0] == "method,alpha,p"
    rows = {(m, round(float(a), 6)): float(p) for m, a, p in (ln.split(",") for ln in prof[1:])}
    assert rows[("A", 1.0)] == 1.0 and rows[("B", 2.9)] == 0.0 and rows[("B", 3.0)] == 1.0
    bad = tmp_path / "bad.txt"
    bad.write_text("3\n1 2 3\n")
    assert cli.main(["logm", str(bad)]) == 2
    assert cli.main(["logm", str(tmp_path / "missing.txt")]) == 2


def test_module_entry_point():
    r = subprocess.run([sys.executable, "-m", "paper_2401_10089_b200", "theta"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("k,order_m,theta")
