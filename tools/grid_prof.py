"""Engine G phase breakdown: LGM_GRID_PROFILE=1 python tools/grid_prof.py --config 4 [--batch B]."""
import argparse
import ctypes
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("LGM_GRID_PROFILE", "1")
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--batch", type=int, default=None)
args = ap.parse_args()
cfg = args.config if args.config in ("3b", "5b") else int(args.config)
lib = _lib.load()
lib.lgm_debug_grid_phase_ms.argtypes = [ctypes.c_void_p, ctypes.c_int]
A = torch.from_numpy(synth.config(cfg, batch=args.batch)).cuda()
opts = driver.LogmOptions(raise_on_error=False)
driver.run_device(A, opts)
torch.cuda.synchronize()
buf = (ctypes.c_double * 8)()
lib.lgm_debug_grid_phase_ms(buf, 1)
t0 = time.perf_counter()
L, rep, ws = driver.run_device(A, opts)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
lib.lgm_debug_grid_phase_ms(buf, 1)
names = ["balance", "alpha(scaling)", "invert", "db_update", "select", "poly", "other"]
print(json.dumps({"config": args.config, "batch": int(A.shape[0]), "wall_ms": wall,
                  "phase_ms": {nm: round(buf[i], 2) for i, nm in enumerate(names)}}, indent=1))
