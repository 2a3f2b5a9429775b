"""Host-side segments of the e2e call (select_and_deform on host arrays,
configs[1]): time spent in each helper per call, wall time of the call, and
the device time of the selection launches. Shows what the host adds around
the device work."""
import sys
import time
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
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


for nm in ("_partition_native", "_partition_device_start", "_boundary_on_device", "_take_buffers", "_give_buffers"):
    wrap(S, nm)
orig_read = S._LoopBuffers.read_all


def read_all(self, then=None):
    t0 = time.perf_counter()
    try:
        return orig_read(self, then)
    finally:
        acc["read_all (incl. wait for the loop)"] += time.perf_counter() - t0


S._LoopBuffers.read_all = read_all
wl = W.config(1)
vol = torch.from_numpy(wl.volume.copy()).pin_memory().numpy()
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)


def step():
    with S._cache_lock:
        S._part_cache.clear()
    t0 = time.perf_counter()
    b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
    acc["BoundarySet()"] += time.perf_counter() - t0
    return P.select_and_deform(b, cfg, vol)


for _ in range(3):
    step()
torch.cuda.synchronize()
acc.clear()
reps = 20
t0 = time.perf_counter()
for _ in range(reps):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / reps
print(f"wall per call {wall * 1e3:.3f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:40s} {v / reps * 1e3:8.3f} ms")
