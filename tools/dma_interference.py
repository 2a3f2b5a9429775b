"""Does a concurrent 48 MB host->device copy slow the one-cluster selection
loop? configs[1] selection timed alone and with the volume's H2D copy issued
on a side stream right before it (device time of the loop launches)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

wl = W.config(1)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m)
pinned = torch.from_numpy(wl.volume.copy()).pin_memory()
dev = torch.empty(pinned.shape, dtype=torch.float64, device="cuda")
side = torch.cuda.Stream()


def sel(with_copy):
    torch.cuda.synchronize()
    if with_copy:
        with torch.cuda.stream(side):
            dev.copy_(pinned, non_blocking=True)
    with N.launch_log(timing=True) as log:
        P.gcb_select(b, cfg)
        torch.cuda.synchronize()
    return sum(log.kernel_ms("rbf_gcb_run"))


sel(False)
out = {"alone_ms": [round(sel(False), 3) for _ in range(5)],
       "with_h2d_ms": [round(sel(True), 3) for _ in range(5)]}
print(out)
