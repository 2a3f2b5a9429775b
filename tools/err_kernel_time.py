"""Time the fused error-scan kernel (rbf_errors_argmax: full-boundary sweep)
on configs[3]'s boundary (Nb = 200k) with Nc supports."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402
from paper_2004_04817_b200.selection import _errors_device  # noqa: E402

wl = W.config(3, nv=1000)
rng = np.random.default_rng(0)
for nc in (300, 1000, 4372):
    idx = rng.choice(wl.nb, nc, replace=False)
    sp, sw = wl.points[idx], rng.normal(size=(nc, 3)) * 1e-3
    b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
    pos = np.arange(wl.nb)
    for _ in range(2):
        _errors_device(pos, b, sp, sw, wl.radius)
    ts = []
    for _ in range(5):
        with N.launch_log(timing=True) as log:
            _errors_device(pos, b, sp, sw, wl.radius)
        ts.append(sum(log.kernel_ms("rbf_errors_argmax")))
    ms = min(ts)
    print(f"Nb {wl.nb} Nc {nc}: {ms:.3f} ms  {22 * wl.nb * nc / (ms * 1e-3) / 1e12:.2f} TFLOP/s algorithmic")
