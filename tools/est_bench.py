"""Estimator micro-benchmark: lgm_est_power_norm_f64 / lgm_est_product_norm_f64 on a batch of
A_I2-like matrices (config-4 shapes), CUDA-event timed; PROG_EST is a plain graph (no
conditional nodes), so ncu can list its kernels.

    python tools/est_bench.py [n=512] [batch=256] [p=7] [product=0]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_10089_b200 import _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
p = int(sys.argv[3]) if len(sys.argv) > 3 else 7
prod = int(sys.argv[4]) if len(sys.argv) > 4 else 0
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 5
lib = _lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))
A = synth.config(4, batch=B, n=n)
A = A / np.abs(A).sum(axis=1).max(axis=1)[:, None, None] * 0.5  # A_I2-like scale
M = torch.from_numpy(A).cuda()
M2 = torch.from_numpy(np.ascontiguousarray(A[:, ::-1, :])).cuda()
est = torch.empty(B, dtype=torch.float64, device="cuda")
ps = torch.empty(B, dtype=torch.int32, device="cuda")
nb = ctypes.c_size_t(0)
lib.lgm_block_workspace_bytes(n, B, ctypes.byref(nb))
ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def run():
    if prod:
        return lib.lgm_est_product_norm_f64(M.data_ptr(), p, M2.data_ptr(), n, B, n, 5, est.data_ptr(), ps.data_ptr(),
                                            ws.data_ptr(), nb.value, s)
    return lib.lgm_est_power_norm_f64(M.data_ptr(), n, B, n, p, 5, est.data_ptr(), ps.data_ptr(), ws.data_ptr(),
                                      nb.value, s)


assert run() == 0
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
passes = ps.cpu().numpy()
gb = passes.sum() * n * n * 8 / 1e9
print(f"n {n} batch {B} p {p} product {prod}: {ms:.3f} ms per estimate, passes mean {passes.mean():.1f}, "
      f"{gb:.1f} GB streamed -> {gb / (ms * 1e-3):.0f} GB/s")
if os.environ.get("EST_OUT"):  # bitwise A/B of estimator paths
    np.savez(os.environ["EST_OUT"], est=est.cpu().numpy(), passes=passes)
