"""Time config-2 logm with an alternative build of the library (A/B experiments).
    LGM_LIB=path python tools/time_lib.py"""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402
_lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))
A = torch.from_numpy(synth.config(int(os.environ.get("CFG", "2")))).cuda()
opts = driver.LogmOptions(raise_on_error=False)
for _ in range(3):
    driver.run_device(A, opts)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L, rep, ws = driver.run_device(A, opts)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
rep = rep.cpu().numpy().view(_lib.REPORT_DTYPE)
print(os.path.basename(os.environ.get("LGM_LIB", "default")), "min ms", round(min(ts), 3), "status ok",
      int((rep["status"] == 0).sum()))
