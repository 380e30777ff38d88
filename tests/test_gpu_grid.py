"""GPU parity for Engine G (n > 64): batched blocked Gauss-Jordan + DMMA GEMMs + batched
estimator, host-orchestrated Algorithm 1.  Same tolerances as tests/test_gpu_parity.py."""
import os

import numpy as np
import pytest

from tests.parity import check_batch, rel_err, tolerance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import paper_2401_10089_b200 as lp  # noqa: E402
from oracle import driver as D  # noqa: E402
from oracle import primitives as P  # noqa: E402
from paper_2401_10089_b200 import constants as C  # noqa: E402
from paper_2401_10089_b200 import synth  # noqa: E402


def test_balance_bitwise_n130(golden):
    A = golden["prim/balance/130/A"]
    B, sc, _ = lp.balance_batched(A)
    assert np.array_equal(B, golden["prim/balance/130/B"])
    assert np.array_equal(sc[0], golden["prim/balance/130/scale"])


@pytest.mark.parametrize("n", [65, 200, 300])
def test_balance_bitwise_vs_oracle(n):
    rng = np.random.default_rng(n)
    d = 2.0 ** rng.integers(-30, 30, n)
    A = rng.standard_normal((2, n, n)) * (d[:, None] / d[None, :])
    B, sc, _ = lp.balance_batched(A)
    for b in range(2):
        Bo, so, _ = P.balance(A[b])
        assert np.array_equal(B[b], Bo) and np.array_equal(sc[b], so)


@pytest.mark.parametrize("n", [65, 100, 257])
@pytest.mark.parametrize("k", [1, 3, 5])
def test_eval_degopt_grid(n, k):
    rng = np.random.default_rng(n + k)
    G = rng.standard_normal((2, n, n))
    X = 0.2 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    c = lp.OpCounter()
    Z = lp.eval_degopt(k, X, counter=c)
    c2 = lp.OpCounter()
    Z2 = lp.eval_degopt(k, X, counter=c2, first_product=X @ X)
    for b in range(2):
        Zo = P.eval_degopt(C.SCHEMES[k - 1], X[b])
        assert rel_err(Z[b], Zo) <= 1e-13
        assert rel_err(Z2[b], Zo) <= 1e-13
    assert c.products == 2 * k and c2.products == 2 * (k - 1)


@pytest.mark.parametrize("n", [65, 130, 300])
@pytest.mark.parametrize("p", [1, 7, 14])
def test_est_power_norm_grid(n, p):
    rng = np.random.default_rng(n * p)
    M = rng.standard_normal((2, n, n)) / np.sqrt(n)
    est, passes = lp.primitives._est(M, p, None, 5, True)
    for b in range(2):
        c = P.Counter()
        v = P.est_power_norm(M[b], p, counter=c)
        assert est[b] == pytest.approx(v, rel=1e-12)
        assert passes[b] == c.estimation_passes


@pytest.mark.parametrize("n", [65, 130])
def test_est_product_norm_grid(n):
    rng = np.random.default_rng(n)
    M1 = rng.standard_normal((2, n, n)) / np.sqrt(n)
    M2 = rng.standard_normal((2, n, n)) / np.sqrt(n)
    est, passes = lp.primitives._est(M1, 7, M2, 5, False)
    for b in range(2):
        c = P.Counter()
        v = P.est_product_norm([(M1[b], 7), (M2[b], 1)], counter=c)
        assert est[b] == pytest.approx(v, rel=1e-12)
        assert passes[b] == c.estimation_passes


def test_est_zero_and_diag_grid():
    Z = np.zeros((1, 80, 80))
    est, passes = lp.primitives._est(Z, 3, None, 5, True)
    assert est[0] == 0.0 and passes[0] == 0
    d = np.linspace(-2, 1.5, 90)
    est, _ = lp.primitives._est(np.diag(d)[None], 3, None, 5, True)
    assert est[0] == pytest.approx(8.0, rel=1e-14)


@pytest.mark.parametrize("n", [65, 128, 200, 320, 384, 512, 520, 545, 1000, 1024])
def test_sqrt_db_grid(n):
    rng = np.random.default_rng(n)
    G = rng.standard_normal((2, n, n))
    A = np.eye(n)[None] + 0.5 * G / np.linalg.norm(G, 2, axis=(1, 2))[:, None, None]
    X, its, st = lp.sqrt_db_batched(A)
    for b in range(2):
        Xo, ito = P.sqrt_db(A[b])
        assert st[b] == 0 and its[b] == ito
        assert rel_err(X[b], Xo) <= 1e-12


def test_sqrt_db_grid_failures():
    n = 70
    A = np.stack([np.diag(np.r_[-1.0, np.linspace(2.0, 3.0, n - 1)]), np.eye(n), np.diag(np.r_[-1.0, np.ones(n - 1)])])
    A[1][3, :] = 0.0
    _, its, st = lp.sqrt_db_batched(A)
    # negative eigenvalue: no convergence; zero row: singular at step 1; diag(-1, 1, ...):
    # X1 = (X0 + I)/2 has an exact zero pivot at step 2 (as in the reference)
    assert list(st) == [2, 1, 1]
    assert list(its) == [50, 0, 1]


def _check(As, L, reps, allow_mismatch=0, allow_stall=0):
    counts, _ = check_batch(As, L, reps, allow_mismatch, allow_stall=allow_stall)
    return counts


@pytest.mark.parametrize("c,n,B", [("3b", 96, 6), (4, 80, 4), ("3b", 128, 4), (2, 100, 6), (3, 72, 2)])
def test_logm_grid_config_shapes(c, n, B):
    A = synth.config(c, batch=B, n=n)
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    _check(A, L, reps, allow_stall=1 if c == 4 else 0)   # (see tests/parity.py db_stall)


def test_logm_grid_near_identity_orders():
    rng = np.random.default_rng(5)
    As = []
    for eps in (1e-12, 1e-8, 1e-5, 1e-3, 2e-2, 0.2):
        G = rng.standard_normal((70, 70))
        As.append(np.eye(70) + eps * G / np.linalg.norm(G, 2))
    As = np.stack(As)
    L, reps = lp.logm_batched(As)
    assert len(set(int(k) for k in reps["k"])) >= 3
    _check(As, L, reps)


def test_logm_grid_identity_and_errors():
    L, rep = lp.logm(np.eye(90))
    assert np.array_equal(L, np.zeros((90, 90))) and (rep.s, rep.k_selected) == (0, 1)
    with pytest.raises(ValueError):
        lp.logm(np.full((70, 70), np.nan))
    with pytest.raises(lp.ConvergenceError):
        lp.logm(np.diag(np.r_[-1.0, np.linspace(2.0, 3.0, 69)]))


def test_logm_grid_spd512_vs_oracle():
    A = synth.config(4, batch=2)
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    _check(A, L, reps)


def test_grid_batches_run_in_passes(tmp_path):
    """Engine G indexes matrices in grid.y/z: batches beyond LGM_GRID_CHUNK (16384) run as
    consecutive passes over one workspace.  A subprocess with LGM_GRID_CHUNK=3 must reproduce
    the single-pass results bit for bit (logm, sqrt_db, balance building blocks)."""
    import os
    import subprocess
    import sys
    A = synth.config("3b", batch=7, n=80)
    np.save(tmp_path / "A.npy", A)
    L1, r1 = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    X1, it1, st1 = lp.sqrt_db_batched(A)
    B1, sc1, sw1 = lp.balance_batched(A)
    code = f"""
import sys, numpy as np
sys.path.insert(0, {repr(ROOT)})
import paper_2401_10089_b200 as lp
A = np.load({repr(str(tmp_path / 'A.npy'))})
L, r = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
X, it, st = lp.sqrt_db_batched(A)
B, sc, sw = lp.balance_batched(A)
np.savez({repr(str(tmp_path / 'out.npz'))}, L=L, r=r.view(np.uint8), X=X, it=it, st=st, B=B, sc=sc, sw=sw)
"""
    env = dict(os.environ, LGM_GRID_CHUNK="3")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    o = np.load(tmp_path / "out.npz")
    assert np.array_equal(o["L"], L1) and o["r"].tobytes() == r1.view(np.uint8).tobytes()
    assert np.array_equal(o["X"], X1) and np.array_equal(o["it"], it1) and np.array_equal(o["st"], st1)
    assert np.array_equal(o["B"], B1) and np.array_equal(o["sc"], sc1) and np.array_equal(o["sw"], sw1)


@pytest.mark.parametrize("c,B", [("3b", 64), (4, 8)])
def test_selection_invariant_grid(c, B):
    """SPEC.md:594 (#7) on Engine G configs: alpha_used <= Theta_k; when s >= 1 the polynomial
    costs exactly k - 1 products (A_I2 reused), k products when s = 0."""
    A = synth.config(c, batch=B)
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    ok = reps["status"] == 0
    assert ok.all()
    th = np.array(C.THETA)[reps["k"] - 1]
    assert (reps["alpha_used"] <= th).all()
    assert (reps["products"] == np.where(reps["s"] >= 1, reps["k"] - 1, reps["k"])).all()



def test_est_fused_matches_per_step_kernels(tmp_path):
    """Engine G's one-launch estimator (est_fused_kernel, n <= 160, M1 in shared memory)
    reproduces the per-step estimator kernels (LGM_EST_FUSED=0, subprocess) bit for bit: the
    estimates, pass counts and the whole logm (reports and L) at config-3b shapes."""
    import subprocess
    import sys
    rng = np.random.default_rng(11)
    mats = {n: rng.standard_normal((3, n, n)) for n in (65, 100, 128, 160)}
    A3 = synth.config("3b", batch=6)
    np.savez(tmp_path / "in.npz", A3=A3, **{f"m{n}": m for n, m in mats.items()})
    ests = {}
    for n, m in mats.items():
        for p, two in ((1, False), (3, True), (7, False)):
            M2 = m[::-1].copy() if two else None
            ests[f"{n}_{p}"] = lp.primitives._est(m, p, M2, 5, True)
    L1, r1 = lp.logm_batched(A3, lp.LogmOptions(raise_on_error=False))
    code = f"""
import sys, numpy as np
sys.path.insert(0, {repr(ROOT)})
import paper_2401_10089_b200 as lp
d = np.load({repr(str(tmp_path / 'in.npz'))})
out = {{}}
for n in (65, 100, 128, 160):
    m = d[f"m{{n}}"]
    for p, two in ((1, False), (3, True), (7, False)):
        e, ps = lp.primitives._est(m, p, m[::-1].copy() if two else None, 5, True)
        out[f"e{{n}}_{{p}}"] = e
        out[f"p{{n}}_{{p}}"] = ps
L, r = lp.logm_batched(d["A3"], lp.LogmOptions(raise_on_error=False))
np.savez({repr(str(tmp_path / 'out.npz'))}, L=L, r=r.view(np.uint8), **out)
"""
    env = dict(os.environ, LGM_EST_FUSED="0")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, timeout=600)
    o = np.load(tmp_path / "out.npz")
    for key, (e, ps) in ests.items():
        assert np.array_equal(o["e" + key], e) and np.array_equal(o["p" + key], ps), key
    assert np.array_equal(o["L"], L1) and o["r"].tobytes() == r1.view(np.uint8).tobytes()


@pytest.mark.parametrize("n,B", [(384, 1), (448, 3)])
def test_logm_grid_g2_small_batches_vs_oracle(n, B):
    """n % 64 == 0, 256 < n <= 512 inverts on the per-panel G2 path (single-CTA panels,
    rank-64 combined passes) whatever the batch size: one and three matrices."""
    A = synth.config(4, batch=B, n=n)
    L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
    _check(A, L, reps)


def test_sqrt_db_g2_small_failures():
    """The G2 single-CTA-panel path (n = 320): a zero row is singular at the first step, an
    eigenvalue on the negative axis does not converge (as in the reference), and a healthy
    matrix in the same batch is unaffected."""
    n = 320
    rng = np.random.default_rng(3)
    G = rng.standard_normal((n, n))
    good = np.eye(n) + 0.5 * G / np.linalg.norm(G, 2)
    zero_row = good.copy()
    zero_row[11, :] = 0.0
    neg = np.diag(np.r_[-1.0, np.linspace(2.0, 3.0, n - 1)])
    X, its, st = lp.sqrt_db_batched(np.stack([good, zero_row, neg]))
    assert list(st) == [0, 1, 2]
    assert its[1] == 0 and its[2] == 50
    Xo, ito = P.sqrt_db(good)
    assert its[0] == ito and rel_err(X[0], Xo) <= 1e-12


def test_grid_call_is_stream_ordered_and_nonblocking():
    """lgm_logm_f64 for n > 64 is one CUDA-graph launch with device-side loops: the host
    call returns while the stream is still busy (no cudaStreamSynchronize anywhere), and the
    result equals the synchronous run bit for bit."""
    import time
    from paper_2401_10089_b200 import _lib, driver
    A = torch.from_numpy(synth.config(4, batch=4, n=256)).cuda()
    opts = lp.LogmOptions(raise_on_error=False)
    s = torch.cuda.current_stream()
    L0, r0, _ = driver.run_device(A, opts, s)                 # capture + instantiate (cached per
    torch.cuda.synchronize()                                  # workspace; the driver reuses it)
    n0 = _lib.launch_count()
    torch.cuda._sleep(3_000_000_000)                          # ~1.5 s of GPU spin ahead of the call
    t0 = time.perf_counter()
    L1, r1, _ = driver.run_device(A, opts, s)
    dt = time.perf_counter() - t0
    assert not s.query()                                      # still queued behind the spin
    torch.cuda.synchronize()
    assert dt < 0.5, dt
    assert torch.equal(L0, L1) and torch.equal(r0, r1)
    assert _lib.launch_count() - n0 > 100                     # kernels executed inside the graph


def test_sharding_bitwise_large_n():
    """a matrix's arithmetic must not depend on its batch-mates (rank-64 / rank-32
    passes chosen by n only).  n = 576 (G2 cluster panels): batch of 3 vs each matrix alone."""
    A = synth.config("5b", batch=3, n=576)
    L3, r3 = lp.logm_batched(A)
    for b in range(3):
        L1, r1 = lp.logm_batched(A[b:b + 1])
        assert np.array_equal(L1[0], L3[b]) and r1.tobytes() == r3[b:b + 1].tobytes()


def test_graph_cache_distinct_workspaces_and_shapes():
    """The per-(workspace, n, batch) graph cache: interleaved calls of different shapes and
    workspaces reproduce their own first results exactly."""
    outs = {}
    for rep in range(2):
        for n, B in ((80, 3), (96, 5), (80, 2)):
            A = synth.config("3b", batch=B, n=n)
            L, r = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
            if rep == 0:
                outs[(n, B)] = (L, r)
            else:
                assert np.array_equal(outs[(n, B)][0], L) and outs[(n, B)][1].tobytes() == r.tobytes()


@pytest.mark.parametrize("n", [80, 320])
def test_grid_concurrent_threads(n):
    """Engine G reentrancy: two host threads (own streams, own workspaces, so two graph-cache
    entries captured and launched concurrently) reproduce their single-thread results."""
    import threading
    A1 = synth.config("3b", batch=6, n=n)
    A2 = synth.config(4, batch=5, n=n)
    ref1, r1 = lp.logm_batched(A1, lp.LogmOptions(raise_on_error=False))
    ref2, r2 = lp.logm_batched(A2, lp.LogmOptions(raise_on_error=False))
    out, err = {}, []

    def run(key, A):
        try:
            for _ in range(3):
                out[key] = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
        except Exception as e:  # noqa: BLE001
            err.append(e)

    ts = [threading.Thread(target=run, args=("a", A1)), threading.Thread(target=run, args=("b", A2))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not err, err
    # (failed matrices -- a config-4 spectrum at small n can stall at the DB noise floor --
    # carry an all-NaN L: compare NaN-aware)
    assert np.array_equal(out["a"][0], ref1, equal_nan=True) and out["a"][1].tobytes() == r1.tobytes()
    assert np.array_equal(out["b"][0], ref2, equal_nan=True) and out["b"][1].tobytes() == r2.tobytes()
