"""Two-rows-per-thread pair panel (gj_panel_pair2_kernel, default for
256 < n <= 512): pivot rule, FMA chains, stage-1 products and the log|det| summation order are
those of gj_panel_pair_kernel<512>, so every bit of L and every report field must equal the
one-row-per-thread kernel's (LGM_PANEL2=0), including the exact-zero-pivot path.
Subprocesses: the switch is read once per process."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2401_10089_b200 import driver, synth, _lib, primitives
out = {}
for cfg, n, b in ((4, 320, 3), (4, 384, 2), (4, 448, 2), (4, 512, 3), ("3b", 512, 2)):
    A = torch.from_numpy(synth.config(cfg, batch=b, n=n)).cuda()
    L, rep, ws = driver.run_device(A, driver.LogmOptions(raise_on_error=False))
    torch.cuda.synchronize()
    r = rep.cpu().numpy().view(_lib.REPORT_DTYPE)[:b]
    out[f"{cfg}_{n}"] = {"L": L.cpu().numpy().view(np.int64).tolist(),
                         "rep": {f: r[f].tolist() for f in ("status", "s", "k", "db_iters", "divisions")}}
# exactly singular input (two equal rows and a zero column): the zero-pivot exit of the panel
A = synth.config(4, batch=2, n=320)
A[1, 7, :] = A[1, 3, :]
A[1, :, 11] = 0.0
X, its, st = primitives.sqrt_db_batched(A)
out["singular"] = {"st": np.asarray(st).tolist(), "its": np.asarray(its).tolist(),
                   "X0": np.asarray(X)[0].view(np.int64).tolist()}
print(json.dumps(out))
""" % ROOT


def _run(**env_over):
    env = dict(os.environ)
    env.pop("LGM_PANEL2", None)
    env.update(env_over)
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_two_row_pair_panel_is_bit_identical():
    one_row = _run(LGM_PANEL2="0")
    two_row = _run()
    for key in one_row:
        assert two_row[key] == one_row[key], key
    assert one_row["singular"]["st"][0] == 0 and one_row["singular"]["st"][1] != 0


G1_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %r)
from paper_2401_10089_b200 import driver, synth, _lib
out = {}
for cfg, n, b in (("3b", 128, 6), ("3b", 96, 4), (3, 128, 2)):
    A = torch.from_numpy(synth.config(cfg, batch=b, n=n)).cuda()
    L, rep, ws = driver.run_device(A, driver.LogmOptions(raise_on_error=False))
    torch.cuda.synchronize()
    r = rep.cpu().numpy().view(_lib.REPORT_DTYPE)[:b]
    out[f"{cfg}_{n}"] = {"L": L.cpu().numpy().view(np.int64).tolist(),
                         "rep": {f: r[f].tolist() for f in ("status", "s", "k", "db_iters", "divisions")}}
print(json.dumps(out))
""" % ROOT


@pytest.mark.gpu
def test_g1_warp_panel_opt_in_is_bit_identical():
    """gj_inv_cta_kernel<128, true> (LGM_G1_WP=1, measured slower and off by default): the
    searched-steps + replay order applies the block panel's FMAs per element in the same order."""
    def run(**env_over):
        env = dict(os.environ)
        env.pop("LGM_G1_WP", None)
        env.update(env_over)
        r = subprocess.run([sys.executable, "-c", G1_SCRIPT], env=env, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        return json.loads(r.stdout.strip().splitlines()[-1])
    block, warp = run(), run(LGM_G1_WP="1")
    for key in block:
        assert warp[key] == block[key], key
