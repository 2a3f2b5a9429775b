"""One warm step of the bench workload (selection + volume deform) for ncu.

    python tools/prof_step.py [--config 1] [--steps 2]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--steps", type=int, default=2)
args = ap.parse_args()
wl = W.config(args.config)
b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
vol = torch.from_numpy(wl.volume).cuda()
for _ in range(args.steps):
    res = P.gcb_select(b, cfg)
    sp = torch.from_numpy(res.support.points).cuda()
    sw = torch.from_numpy(res.support.weights).cuda()
    out = P.eval_device(vol, sp, sw, wl.radius, deform=True)
torch.cuda.synchronize()
print("Nc", len(res.support), "iterations", len(res.history.records))
