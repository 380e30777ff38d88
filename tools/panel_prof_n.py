"""clock64 phases of the G2 panel kernels through the inversion micro-benchmark entry (debug build):
    make gvariant V=pp VFLAGS=-DLGM_PANEL_PROF
    LGM_LIB=paper_2401_10089_b200/_build/var/liblogmpoly_b200_pp.so python tools/panel_prof_n.py [n=4096] [batch=8]
n > 512: gj_panel_cluster_kernel (per CTA of the 8-CTA cluster); 256 < n <= 512: the pair panel."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2401_10089_b200 import _lib, synth
n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
lib = _lib.load(os.environ["LGM_LIB"])
lib.lgm_debug_invert_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]
A = torch.from_numpy(synth.config(4, batch=B, n=n)).cuda()
wsb = ctypes.c_size_t(0)
lib.lgm_workspace_bytes(n, B, ctypes.byref(wsb))
ws = torch.empty(wsb.value, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
rc = lib.lgm_debug_invert_f64(A.data_ptr(), n, B, 1, ws.data_ptr(), ctypes.c_void_p(s.cuda_stream))
torch.cuda.synchronize()
assert rc == 0, rc
buf = (ctypes.c_ulonglong * 12)()
lib.lgm_debug_panel_cycles(buf)
v = list(buf); c = max(v[4], 1)
print("n", n, "panel CTAs", c, "cycles/CTA: load %.0f factor %.0f store %.0f" % (v[0] / c, v[2] / c, v[3] / c))
if n <= 256:  # G1: per 32-column panel of gj_inv_cta_kernel
    print("G1 per panel: load %.0f  32 pivot steps %.0f  store+stage+first snapshot %.0f  trailing update %.0f" %
          (v[0] / c, v[2] / c, v[3] / c, v[1] / c))
    sys.exit(0)
print("per pivot step: search+block barrier %.0f  candidate publish %.0f  cluster barrier %.0f  winner fetch+barrier %.0f"
      % (v[6] / c / 32, v[9] / c / 32, v[7] / c / 32, v[10] / c / 32))
