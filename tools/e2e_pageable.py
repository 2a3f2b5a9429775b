"""deform_points on a host volume: pinned vs pageable numpy input (the
reference API callers pass pageable arrays), and the cost of page-locking a
pageable array in place (cudaHostRegister). configs[1] support set.

    python tools/e2e_pageable.py [--nv 2000000] [--reps 10]
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nv", type=int, default=2_000_000)
ap.add_argument("--reps", type=int, default=10)
args = ap.parse_args()
wl = W.config(1, nv=args.nv)
res = P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp),
                   P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m))
sup = res.support
pageable = np.ascontiguousarray(wl.volume)
pinned = torch.from_numpy(pageable.copy()).pin_memory().numpy()


def timed(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * float(np.median(ts))


out = {}
out["pinned_ms"] = timed(lambda: P.deform_points(pinned, sup, wl.radius))
out["pageable_ms"] = timed(lambda: P.deform_points(pageable, sup, wl.radius))
cudart = torch.cuda.cudart()


def reg():
    a = np.empty_like(pageable)
    t0 = time.perf_counter()
    cudart.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    t1 = time.perf_counter()
    cudart.cudaHostUnregister(a.ctypes.data)
    return t1 - t0


reg()
out["host_register_48MB_ms"] = 1e3 * float(np.median([reg() for _ in range(5)]))
a = np.empty_like(pageable)
t0 = time.perf_counter()
np.copyto(a, pageable)
out["memcpy_48MB_ms"] = 1e3 * (time.perf_counter() - t0)
print(out)
