"""Engine G inversion micro-benchmark: 2*batch Gauss-Jordan inversions of n x n matrices
(config-4 SPD inputs), timed with CUDA events around lgm_debug_invert_f64 (direct launches,
so ncu can profile every kernel).

    python tools/inv_bench.py [n=512] [batch=256] [reps=5]
Prints ms per DB-step-equivalent (2*batch inversions) and the algorithmic FP64 TFLOP/s
(2 n^3 per inversion) against the measured DMMA peak.
"""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2401_10089_b200 import _lib, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
lib = _lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))  # LGM_LIB: A/B variant builds (make gvariant)
lib.lgm_debug_invert_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]
A = torch.from_numpy(synth.config(4, batch=B, n=n)).cuda()
wsb = ctypes.c_size_t(0)
lib.lgm_workspace_bytes(n, B, ctypes.byref(wsb))
ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
rc = lib.lgm_debug_invert_f64(A.data_ptr(), n, B, 1, ws.data_ptr(), ctypes.c_void_p(s.cuda_stream))
assert rc == 0, rc
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
rc = lib.lgm_debug_invert_f64(A.data_ptr(), n, B, reps, ws.data_ptr(), ctypes.c_void_p(s.cuda_stream))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
tf = 2 * B * 2.0 * n ** 3 / (ms * 1e-3) / 1e12
print(f"n {n} jobs {2 * B}: {ms:.3f} ms per step, {tf:.2f} TFLOP/s ({100 * tf / 36.945:.1f}% of DMMA peak)")
