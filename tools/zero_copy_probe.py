"""Volume kernel reading its targets from and writing its results to pinned
host memory directly (zero-copy over PCIe, UVA-mapped pinned buffers) vs the
device-resident launch and vs the chunked copy pipeline (rbf_eval_host).
configs[1] support set, 2M targets.

    python tools/zero_copy_probe.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

wl = W.config(1)
res = P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp),
                   P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m))
lib = N.load()
sp = torch.from_numpy(res.support.points).cuda()
sw = torch.from_numpy(res.support.weights).cuda()
n = wl.nv
host_in = torch.from_numpy(wl.volume.copy()).pin_memory()
host_out = torch.empty((n, 3), dtype=torch.float64).pin_memory()
dev_in = host_in.cuda()
dev_out = torch.empty_like(dev_in)


def run(src, dst):
    rc = lib.rbf_eval(src.data_ptr(), n, sp.data_ptr(), sw.data_ptr(), sp.shape[0], wl.radius, 1,
                      dst.data_ptr(), N.stream_ptr())
    N.check(rc, "rbf_eval")


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


out = {"device_ms": timed(lambda: run(dev_in, dev_out)),
       "zero_copy_in_out_ms": timed(lambda: run(host_in, host_out)),
       "zero_copy_out_only_ms": timed(lambda: run(dev_in, host_out)),
       "pipeline_ms": timed(lambda: P.deform_points(host_in.numpy(), res.support, wl.radius))}
run(host_in, host_out)
torch.cuda.synchronize()
ref = dev_out.cpu().numpy()
run(dev_in, dev_out)
torch.cuda.synchronize()
out["zero_copy_equal"] = bool(np.array_equal(host_out.numpy(), dev_out.cpu().numpy()))
print(out)
