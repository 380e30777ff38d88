"""Engine G phase split from the device-side phase timer (lgm_debug_grid_phase_ns):

    python tools/grid_phases.py [config=4] [batch]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402

NAMES = ["load", "balance", "alpha (scaling)", "DB (inversion+update)", "select prep", "select", "poly", "other"]
cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
cfg = cfg if cfg in ("3b", "5b") else int(cfg)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
A = torch.from_numpy(synth.config(cfg, batch=batch)).cuda()
opts = lp.LogmOptions(raise_on_error=False)
lib = _lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))  # LGM_LIB: A/B builds
lib.lgm_debug_grid_phase_ns.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
driver.run_device(A, opts)
torch.cuda.synchronize()
lib.lgm_debug_grid_phase_ns(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3
e0.record()
for _ in range(reps):
    driver.run_device(A, opts)
e1.record()
torch.cuda.synchronize()
lib.lgm_debug_grid_phase_ns(buf, 1)
tot = sum(buf)
print(f"config {cfg} {tuple(A.shape)}: {e0.elapsed_time(e1) / reps:.2f} ms per call (events)")
for nm, v in zip(NAMES, buf):
    print(f"  {nm:24s} {v / reps / 1e6:9.2f} ms  {100.0 * v / max(tot, 1):5.1f}%")
