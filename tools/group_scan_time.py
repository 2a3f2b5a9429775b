"""Time group_arg_max_error's device scan (rbf_errors_argmax) on GCB-sized
groups: rows x supports of configs 1-3's groups."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200.selection import _errors_device  # noqa: E402

rng = np.random.default_rng(0)
for nb, card, nc in ((20_000, 625, 287), (80_000, 1667, 848), (200_000, 3125, 4372), (200_000, 200_000, 4372)):
    pts = rng.uniform(-1, 1, (nb, 3))
    b = P.stage_boundary(P.BoundarySet(np.arange(nb), pts, rng.normal(size=(nb, 3)) * 1e-2))
    sp, sw = pts[:nc], rng.normal(size=(nc, 3)) * 1e-3
    pos = rng.choice(nb, card, replace=False)
    for _ in range(3):
        _errors_device(pos, b, sp, sw, 2.0)
    ts = []
    for _ in range(7):
        with N.launch_log(timing=True) as log:
            _errors_device(pos, b, sp, sw, 2.0)
        ts.append(sum(log.kernel_ms("rbf_errors_argmax")))
    ms = min(ts)
    print(f"rows {card:6d} x supports {nc:5d}: {ms * 1e3:8.1f} us  {22 * card * nc / (ms * 1e-3) / 1e12:6.2f} TFLOP/s")
