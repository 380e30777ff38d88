"""Out-of-bounds write check on the GPU (compute-sanitizer is closed on this pool): every
logm engine path, failure path and building block runs with 4 KiB guard bands after each
workspace region and n x n slot (LGM_WS_GUARD=1) and canary pads around every output; no
guard or canary byte may change, and the guarded run (different slot strides) must give the
same bits as the unguarded one."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _probe(out, guard):
    env = dict(os.environ)
    env.pop("LGM_WS_GUARD", None)
    if guard:
        env["LGM_WS_GUARD"] = "1"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "guard_probe.py"), str(out)], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_workspace_guard_bands_and_output_canaries(tmp_path):
    out = _probe(tmp_path / "g.npz", True)
    assert out["selftest_detected"] == 3, out["selftest_detected"]  # the checker sees poked guard bytes
    res = out["calls"]
    assert len(res) >= 30
    assert all(r["guarded"] for r in res), "LGM_WS_GUARD=1 did not enable the guard bands"
    bad = [r for r in res if r["rc"] != 0 or r["bad"] != 0 or not r["canary"]]
    assert not bad, bad
    ref = _probe(tmp_path / "u.npz", False)["calls"]
    assert not any(r["guarded"] for r in ref)
    a, b = np.load(tmp_path / "g.npz"), np.load(tmp_path / "u.npz")
    assert sorted(a.files) == sorted(b.files)
    diff = [k for k in a.files if not np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8))]
    assert not diff, diff
