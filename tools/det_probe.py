"""Determinism probe: the same batch through fresh workspaces / streams / threads must give
identical bits (reports and L).  Prints which fields differ."""
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 80
A = torch.from_numpy(synth.config(4, batch=5, n=n)).cuda()
opts = lp.LogmOptions(raise_on_error=False)


def run(stream):
    L, rep, ws = driver.run_device(A, opts, stream)
    torch.cuda.synchronize()
    return L.cpu().numpy(), rep.cpu().numpy().view(_lib.REPORT_DTYPE)[:5].copy()


def cmp(tag, a, b):
    La, ra = a
    Lb, rb = b
    diff = [f for f in _lib.REPORT_DTYPE.names if not np.array_equal(ra[f], rb[f])]
    print(tag, "L equal", np.array_equal(La, Lb), "max |dL|", float(np.abs(La - Lb).max()), "report fields differing", diff,
          flush=True)
    if diff:
        for f in diff:
            print("   ", f, ra[f], rb[f])


s0 = torch.cuda.current_stream()
base = run(s0)
cmp("same stream again", base, run(s0))
s1 = torch.cuda.Stream()
cmp("new stream (new workspace)", base, run(s1))
s2 = torch.cuda.Stream()
cmp("another new stream", base, run(s2))
res = {}


def th(key):
    s = torch.cuda.Stream()
    for _ in range(3):
        res[key] = run(s)


ts = [threading.Thread(target=th, args=(k,)) for k in ("a", "b")]
B2 = torch.from_numpy(synth.config("3b", batch=6, n=n)).cuda()
for t in ts:
    t.start()
for _ in range(3):
    driver.run_device(B2, opts, torch.cuda.current_stream())
for t in ts:
    t.join()
cmp("thread a", base, res["a"])
cmp("thread b", base, res["b"])
