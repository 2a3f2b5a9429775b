"""Host-side time per segment of gcb_select on configs[1] (wraps the
selection module's helpers; the remainder is readback + record building)."""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import selection as S  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

acc = defaultdict(float)


def wrap(mod, name):
    fn = getattr(mod, name)

    def inner(*a, **k):
        t0 = time.perf_counter()
        try:
            return fn(*a, **k)
        finally:
            acc[name] += time.perf_counter() - t0

    setattr(mod, name, inner)


for nm in ("_partition_positions", "_boundary_on_device", "_to_device", "_read_state", "_LoopBuffers",
           "SupportSet", "IterationRecord"):
    wrap(S, nm)

wl = W.config(1, nv=1000)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
for _ in range(3):
    P.gcb_select(b, cfg)
torch.cuda.synchronize()
acc.clear()
N = 20
t0 = time.perf_counter()
for _ in range(N):
    P.gcb_select(b, cfg)
torch.cuda.synchronize()
total = (time.perf_counter() - t0) / N
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"{k:24s} {v / N * 1e3:8.3f} ms")
print(f"{'total per call':24s} {total * 1e3:8.3f} ms")
