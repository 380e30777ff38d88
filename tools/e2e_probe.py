"""Probe the host-buffer path: wall time of logm_batched per chunk count (config 2).

    python tools/e2e_probe.py [--config 2]
"""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import driver, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="2")
args = ap.parse_args()
cfg = args.config if args.config in ("3b", "5b") else int(args.config)
A = synth.config(cfg)
Ah = torch.from_numpy(A).pin_memory()
opts = lp.LogmOptions(raise_on_error=False)
orig = driver._host_chunks
Ad = Ah.cuda()
for _ in range(3):
    driver.run_device(Ad, opts)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    driver.run_device(Ad, opts)
torch.cuda.synchronize()
print(f"device-resident run_device: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
for nc in (1, 2, 3, 4, 6, 8):
    driver._host_chunks = lambda B, n, nc=nc: nc
    Lo = torch.empty_like(Ah).pin_memory()
    for _ in range(3):
        lp.logm_batched(Ah, opts, out=Lo)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        lp.logm_batched(Ah, opts, out=Lo)
        ts.append(time.perf_counter() - t0)
    ts.sort()
    print(f"chunks={nc}: median {ts[len(ts) // 2] * 1e3:.3f} ms  min {ts[0] * 1e3:.3f} ms")
driver._host_chunks = orig
# pure copy costs
x = torch.empty_like(Ad)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    x.copy_(Ah, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D {A.nbytes / 1e6:.1f} MB: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
Lh = torch.empty_like(Ah).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    Lh.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"D2H: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
t0 = time.perf_counter()
for _ in range(10):
    torch.empty((4096, 32, 32), dtype=torch.float64, pin_memory=True)
print(f"pinned alloc: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
