"""One logm_batched device run of a config (for ncu captures): python tools/run_once.py --config 4"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2401_10089_b200 import driver, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--batch", type=int, default=None)
args = ap.parse_args()
cfg = args.config if args.config in ("3b", "5b") else int(args.config)
A = torch.from_numpy(synth.config(cfg, batch=args.batch)).cuda()
L, rep, ws = driver.run_device(A, driver.LogmOptions(raise_on_error=False))
torch.cuda.synchronize()
print("ok")
