"""Does an Engine G call block the host?  Times each step of a call issued behind a ~1.5 s
GPU spin, for a cached graph (same workspace) and a new workspace (graph capture)."""
import ctypes
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2401_10089_b200 as lp  # noqa: E402
from paper_2401_10089_b200 import _lib, driver, synth  # noqa: E402

A = torch.from_numpy(synth.config(4, batch=4, n=256)).cuda()
opts = lp.LogmOptions(raise_on_error=False)
lib = _lib.load()
wsb = ctypes.c_size_t(0)
lib.lgm_workspace_bytes(256, 4, ctypes.byref(wsb))
wss = [torch.empty(wsb.value, dtype=torch.uint8, device=A.device) for _ in range(3)]
L = torch.empty_like(A)
rep = torch.empty(4 * 64, dtype=torch.uint8, device=A.device)
o, keep = driver._c_opts(opts)
s = torch.cuda.current_stream()
for trial, wi in enumerate([0, 0, 1, 2, 1]):
    torch.cuda.synchronize()
    torch.cuda._sleep(3_000_000_000)
    t0 = time.perf_counter()
    rc = lib.lgm_logm_f64(A.data_ptr(), L.data_ptr(), 256, 4, 256, ctypes.byref(o), rep.data_ptr(),
                          wss[wi].data_ptr(), wsb.value, ctypes.c_void_p(s.cuda_stream))
    t1 = time.perf_counter()
    print(trial, "ws", wi, "rc", rc, "call %.3f ms" % ((t1 - t0) * 1e3), "busy", not s.query(), flush=True)
torch.cuda.synchronize()
