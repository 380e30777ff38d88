"""Per-phase clock64 cycles of gj_panel_cta_kernel (G2 for n <= 512; debug build):
    make gvariant V=pp VFLAGS=-DLGM_PANEL_PROF && LGM_G1_MAXN=0 LGM_LIB=paper_2401_10089_b200/_build/var/liblogmpoly_b200_pp.so python tools/panel_prof.py"""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2401_10089_b200 import _lib, driver, synth
lib = _lib.load(os.environ["LGM_LIB"])
A = torch.from_numpy(synth.config(4)).cuda()
driver.run_device(A, driver.LogmOptions(raise_on_error=False)); torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 12)()
lib.lgm_debug_panel_cycles(buf)
v = list(buf); c = v[4]
print("CTAs", c, "cycles/CTA: load %.0f stage1 %.0f factor %.0f store %.0f" % tuple(x / c for x in v[:4]))
if v[6]:  # two-rows-per-thread panel: per pivot step (32 per panel)
    print("panel2 cycles/step: search+barrier %.0f  winner+rcp+publish+barrier %.0f  row loads+FMAs %.0f" %
          tuple(x / c / 32 for x in v[6:9]))
