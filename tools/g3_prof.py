"""G3 phase cycles (debug build with -DLGM_G3_PROF: make gvariant V=g3prof VFLAGS=-DLGM_G3_PROF):
    LGM_G3=1 LGM_LIB=paper_2401_10089_b200/_build/var/liblogmpoly_b200_g3prof.so python tools/g3_prof.py [n] [batch]"""
import ctypes
import os
import sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2401_10089_b200 import _lib, synth  # noqa: E402
n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
B = int(sys.argv[2]) if len(sys.argv) > 2 else 256
lib = _lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))
lib.lgm_debug_invert_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
A = torch.from_numpy(synth.config(4, batch=B, n=n)).cuda()
wsb = ctypes.c_size_t(0)
lib.lgm_workspace_bytes(n, B, ctypes.byref(wsb))
ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
out = (ctypes.c_ulonglong * 8)()
lib.lgm_debug_invert_f64(A.data_ptr(), n, B, 1, ws.data_ptr(), s)
torch.cuda.synchronize()
lib.lgm_debug_g3_cycles(out, 1)
lib.lgm_debug_invert_f64(A.data_ptr(), n, B, 1, ws.data_ptr(), s)
torch.cuda.synchronize()
lib.lgm_debug_g3_cycles(out, 0)
jobs = 2 * B
names = ["P wait narrow", "P panels", "U wait panel", "U W formation", "U narrow tiles", "U other tiles"]
for i, nm in enumerate(names):
    print(f"{nm:16s} {out[i] / jobs / 1e3:9.1f} kcycles per job")
