"""cProfile of gcb_select on an unstaged numpy boundary (configs[1]): where the
host time between the API call and the device loop goes."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

wl = W.config(1, nv=1000)
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)


def step():
    return P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp), cfg)


for _ in range(5):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(22)
