"""cProfile of the bench step (gcb_select on a staged boundary + volume
eval) to expose host-side overheads."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

wl = W.config(1)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
vol = torch.from_numpy(wl.volume).cuda()
out = torch.empty_like(vol)


def step():
    res = P.gcb_select(b, cfg)
    sp = torch.from_numpy(res.support.points).cuda()
    sw = torch.from_numpy(res.support.weights).cuda()
    P.eval_device(vol, sp, sw, wl.radius, deform=True, out=out)
    return res


for _ in range(3):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    step()
torch.cuda.synchronize()
print("wall ms/step", (time.perf_counter() - t0) * 100)
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
