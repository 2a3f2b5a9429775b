"""One greedy (m=1) selection on the configs[2] boundary (Nb = 80k): the
error-scan showcase of BASELINE configs[4]; used for ncu captures."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2004_04817_b200 as P
from paper_2004_04817_b200 import workloads as W

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cap = int(sys.argv[2]) if len(sys.argv) > 2 else None
wl = W.config(2, nv=1000)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=cap or wl.nb, m=m, seed=0)
r = P.gcb_select(b, cfg)
torch.cuda.synchronize()
print(len(r.support))
