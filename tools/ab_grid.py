"""A/B one BASELINE config across library variants: time logm (device path) and compare L /
reports against the first library (run in separate processes: one library per process).

    python tools/ab_grid.py CFG BATCH lib1.so[:VAR=val,...] lib2.so ...
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    _, _, cfg, batch, lib, out = sys.argv
    sys.path.insert(0, ROOT)
    import torch  # noqa: E402
    from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402
    _lib.load(lib)
    cfg = cfg if cfg in ("3b", "5b") else int(cfg)
    A = torch.from_numpy(synth.config(cfg, batch=int(batch))).cuda()
    opts = driver.LogmOptions(raise_on_error=False)
    driver.run_device(A, opts)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record()
        L, rep, ws = driver.run_device(A, opts)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    np.savez(out, L=L.cpu().numpy(), rep=rep.cpu().numpy(), ms=np.array(ts))
    sys.exit(0)

cfg, batch, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
base = None
for i, lib in enumerate(libs):
    out = f"/tmp/ab_{i}.npz"
    env = dict(os.environ)
    path, _, kv = lib.partition(":")  # lib.so[:VAR=val,VAR2=val]
    for item in filter(None, kv.split(",")):
        k, _, v = item.partition("=")
        env[k] = v
    r = subprocess.run([sys.executable, __file__, "--one", cfg, batch, path, out], capture_output=True, text=True,
                       env=env)
    if r.returncode:
        print(os.path.basename(lib), "FAILED", r.stderr[-2000:])
        continue
    d = np.load(out)
    rep = d["rep"].view(np.dtype([("status", "<i4"), ("s", "<i4"), ("k", "<i4"), ("db_iters", "<i4"),
                                  ("rest", "<i4", (8,)), ("alpha", "<f8"), ("mm", "<f8")]))
    msg = f"{os.path.basename(lib)}: {min(d['ms']):.2f} ms (min of 3)"
    if base is None:
        base = (d["L"], rep)
    else:
        L0, r0 = base
        ok = np.isfinite(L0).all(axis=(1, 2)) & np.isfinite(d["L"]).all(axis=(1, 2))
        num = np.linalg.norm((d["L"] - L0)[ok], axis=(1, 2))
        den = np.linalg.norm(L0[ok], axis=(1, 2))
        rel = float((num / den).max()) if ok.any() else 0.0
        same = {f: int((rep[f] == r0[f]).sum()) for f in ("status", "s", "k", "db_iters")}
        msg += f"  max rel dL vs first {rel:.2e}  equal {same} of {len(rep)}"
    print(msg, flush=True)
