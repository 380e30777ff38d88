"""Time one config through logm_batched device path with an alternative library (A/B).
    LGM_LIB=path CFG=5b BATCH=8 python tools/time_grid.py"""
import os
import sys
import time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402
_lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))
cfg = os.environ.get("CFG", "5b")
cfg = cfg if cfg in ("3b", "5b") else int(cfg)
b = os.environ.get("BATCH")
A = torch.from_numpy(synth.config(cfg, batch=int(b) if b else None)).cuda()
opts = driver.LogmOptions(raise_on_error=False)
driver.run_device(A, opts)
torch.cuda.synchronize()
ts = []
for _ in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    L, rep, ws = driver.run_device(A, opts)
    torch.cuda.synchronize()
    ts.append(time.perf_counter() - t0)
rep = rep.cpu().numpy().view(_lib.REPORT_DTYPE)
print(os.path.basename(os.environ.get("LGM_LIB", "default")), cfg, "min ms", round(min(ts) * 1e3, 1),
      "statuses", sorted(set(rep["status"].tolist())))
