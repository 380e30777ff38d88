"""One logm call on a BASELINE config (device-resident input), for ncu launch lists:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file out.csv \
        python tools/prof_one.py 4 [batch]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import driver, synth  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "4"
cfg = cfg if cfg in ("3b", "5b") else int(cfg)
batch = int(sys.argv[2]) if len(sys.argv) > 2 else None
A = torch.from_numpy(synth.config(cfg, batch=batch)).cuda()
L, rep, ws = driver.run_device(A, lp.LogmOptions(raise_on_error=False))
torch.cuda.synchronize()
print("done", A.shape)
