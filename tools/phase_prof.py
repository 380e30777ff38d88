"""Per-phase cycle breakdown of the fused kernel (debug build with -DLGM_PHASE_PROF).

    make prof && python tools/phase_prof.py [--config 2] [--batch 4096]
Prints the share of CTA-cycles (thread 0 clock64 deltas summed over CTAs) per Algorithm-1
phase: balance, scaling-loop alpha (norm estimation), sqrt_db, select, polynomial.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
ap.add_argument("--batch", type=int, default=None)
args = ap.parse_args()
cfg = args.config if args.config in ("3b", "5b") else int(args.config)
_lib.load(os.environ.get("LGM_PROF_LIB", os.path.join(ROOT, "paper_2401_10089_b200", "_build",
                                                      "liblogmpoly_b200_prof.so")))
lib = _lib._lib
lib.lgm_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
A = torch.from_numpy(synth.config(cfg, batch=args.batch)).cuda()
opts = driver.LogmOptions(raise_on_error=False)
driver.run_device(A, opts)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 8)()
lib.lgm_debug_phase_cycles(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
driver.run_device(A, opts)
e1.record()
torch.cuda.synchronize()
lib.lgm_debug_phase_cycles(buf, 1)
names = ["balance", "alpha(scaling loop)", "sqrt_db", "select", "poly+epilogue",
         "  of which estimator applies (alpha+select)", "  of which estimate() total (alpha+select)", "  of which GJ inversion (sqrt_db, team 0)"]
tot = sum(buf[i] for i in range(5))
out = {"config": args.config, "batch": int(A.shape[0]), "kernel_ms": e0.elapsed_time(e1),
       "cycles_per_matrix": {nm: buf[i] / A.shape[0] for i, nm in enumerate(names)},
       "share": {nm: buf[i] / tot for i, nm in enumerate(names)}}
print(json.dumps(out, indent=1))
