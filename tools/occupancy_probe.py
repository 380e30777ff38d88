"""Engine F latency vs throughput probe: time config-2 batches of 148 x {1, 2, 4, 8, 16, 28} matrices.

    python tools/occupancy_probe.py
At batch 148 every SM holds one CTA (pure per-matrix latency); the per-CTA time at larger
batches shows how much the SM's shared issue / pipes stretch each matrix.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_10089_b200 import driver, synth  # noqa: E402

opts = driver.LogmOptions(raise_on_error=False)
A_all = torch.from_numpy(synth.config(2)).cuda()
for per_sm in (1, 2, 4, 8, 16, 27):
    B = min(148 * per_sm, A_all.shape[0])
    A = A_all[:B].contiguous()
    for _ in range(2):
        driver.run_device(A, opts)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        driver.run_device(A, opts)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    waves = per_sm / 8.0
    print(f"batch {B:5d} ({per_sm:2d}/SM): {t:.3f} ms, {B / t * 1e3:.0f} matrices/s, "
          f"per-CTA time if {min(per_sm, 8)} resident/SM: {t / max(1.0, waves):.3f} ms")
