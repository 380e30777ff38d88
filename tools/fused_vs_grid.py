import os, sys, torch
sys.path.insert(0, '.')
from paper_2401_10089_b200 import _lib, driver, synth
_lib.load(os.environ.get("LGM_LIB", _lib.LIB_PATH))
import numpy as np
for n, B in ((48, 4096), (64, 4096), (64, 1024)):
    A = torch.from_numpy(synth.config(2, batch=B, n=n)).cuda()
    opts = driver.LogmOptions(raise_on_error=False)
    driver.run_device(A, opts); torch.cuda.synchronize()
    import time
    ts=[]
    for _ in range(3):
        t0=time.perf_counter(); driver.run_device(A, opts); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    print(os.path.basename(os.environ.get("LGM_LIB","default")), n, B, round(min(ts)*1e3,2), "ms")
