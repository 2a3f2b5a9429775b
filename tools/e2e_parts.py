"""Wall-time split of the e2e step on configs[1]: gcb_select on an unstaged
boundary, deform_points on a pinned host volume (chunked pipeline), and the
device-resident equivalents."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import core as C  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

wl = W.config(1)
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
vol = torch.from_numpy(wl.volume).pin_memory().numpy()
vol_d = torch.from_numpy(wl.volume).cuda()


def timed(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


res = P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp), cfg)
sup = res.support
print("gcb_select (unstaged)   %.3f ms" % timed(lambda: P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp), cfg)))
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
print("gcb_select (staged)     %.3f ms" % timed(lambda: P.gcb_select(b, cfg)))
print("deform_points (pinned)  %.3f ms" % timed(lambda: P.deform_points(vol, sup, wl.radius)))
vol_pageable = np.array(wl.volume)
print("deform_points (pageable) %.3f ms" % timed(lambda: P.deform_points(vol_pageable, sup, wl.radius)))
sp, sw = torch.from_numpy(sup.points).cuda(), torch.from_numpy(sup.weights).cuda()
out = torch.empty_like(vol_d)
print("eval_device (resident)  %.3f ms" % timed(lambda: P.eval_device(vol_d, sp, sw, wl.radius, deform=True, out=out)))
for chunks in (4, 6, 8, 12, 16, 24, 32):
    C._PIPELINE_CHUNKS = chunks
    print("pipelined, %2d chunks    %.3f ms" % (chunks, timed(lambda: P.deform_points(vol, sup, wl.radius))))
h = torch.empty((wl.nv, 3), dtype=torch.float64, pin_memory=True)
print("H2D 48 MB pinned        %.3f ms" % timed(lambda: vol_d.copy_(torch.from_numpy(vol), non_blocking=True)))
print("D2H 48 MB pinned        %.3f ms" % timed(lambda: h.copy_(vol_d, non_blocking=True)))

# duplex: H2D and D2H of 48 MB each on two streams at once
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
vol_d2 = torch.empty_like(vol_d)
src = torch.from_numpy(vol)


def duplex():
    with torch.cuda.stream(s1):
        vol_d2.copy_(src, non_blocking=True)
    with torch.cuda.stream(s2):
        h.copy_(vol_d, non_blocking=True)
    s1.synchronize()
    s2.synchronize()


print("H2D || D2H 48 MB each   %.3f ms" % timed(duplex))
