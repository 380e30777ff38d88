"""Sanity of the large-n path: logm of config 5b (n=4096) vs expm round trip on the GPU."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2401_10089_b200 as lp
from paper_2401_10089_b200 import synth
cfg = sys.argv[1] if len(sys.argv) > 1 else "5b"
cfg = cfg if cfg in ("3b", "5b") else int(cfg)
n = int(sys.argv[2]) if len(sys.argv) > 2 else None
A = torch.from_numpy(synth.config(cfg, batch=1, n=n)).cuda()
L, reps = lp.logm_batched(A, lp.LogmOptions(raise_on_error=False))
print({k: reps[0][k].item() for k in reps.dtype.names})
if reps[0]["status"] == 0:
    E = torch.linalg.matrix_exp(L)
    print("round trip ||expm(L)-A||_F/||A||_F =", (torch.linalg.matrix_norm(E - A) / torch.linalg.matrix_norm(A)).item())
