"""cProfile of gcb_select on the bench workload (host-side overheads)."""
import cProfile, pstats, sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P
from paper_2004_04817_b200 import workloads as W
wl = W.config(1, nv=1000)
b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
for _ in range(3):
    P.gcb_select(b, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    P.gcb_select(b, cfg)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
