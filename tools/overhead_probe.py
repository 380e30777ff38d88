"""Host overhead of the public API: run_device vs logm_batched on device and host input."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import driver, synth  # noqa: E402

A = synth.config(2)
Ad = torch.from_numpy(A).cuda()
Ah = torch.from_numpy(A).pin_memory()
out = torch.empty_like(Ah).pin_memory()
opts = lp.LogmOptions(raise_on_error=False)


def t(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e3


print("run_device (device in/out)      %.3f ms" % t(lambda: driver.run_device(Ad, opts)))
print("logm_batched device tensor       %.3f ms" % t(lambda: lp.logm_batched(Ad, opts)))
print("logm_batched pinned host + out   %.3f ms" % t(lambda: lp.logm_batched(Ah, opts, out=out)))
# host-side cost of one run_device call without waiting for the GPU
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    driver._c_opts(opts)
print("_c_opts per call                 %.1f us" % ((time.perf_counter() - t0) / 50 * 1e6))
