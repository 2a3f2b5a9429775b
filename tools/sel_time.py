"""Selection-only timing on a BASELINE config's boundary (no volume): one warm
gcb_select, then `reps` timed ones; device ms of the selection launches, t1 / t2
sums, the device phase split (one extra run with RBF_GCB_PHASES) and a hash of
the support sequence (A/B: identical sequences).

    python tools/sel_time.py [--config 3] [--reps 2] [--m M]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402
from paper_2004_04817_b200.selection import _gcb_run  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--m", type=int, default=None)
args = ap.parse_args()
wl = W.config(args.config, nv=16)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=args.m or wl.m, seed=0)
P.gcb_select(b, cfg)
dev = []
for _ in range(args.reps):
    with N.launch_log(timing=True) as log:
        r = P.gcb_select(b, cfg)
        torch.cuda.synchronize()
    dev.append(sum(log.kernel_ms("rbf_gcb_run")))
h = r.history
ph = _gcb_run(b, cfg, phases=True).history.device_phase_cycles
print(json.dumps({"config": args.config, "m": cfg.m, "nc": len(r.support), "iterations": len(h.records),
                  "dev_ms": [round(x, 3) for x in dev], "t1_ms": round(1e3 * sum(x.t1_s for x in h.records), 3),
                  "t2_ms": round(1e3 * sum(x.t2_s for x in h.records), 3),
                  "phases_us": {k: round(v / 1.965e3, 1) for k, v in ph.items() if v},
                  "seq_hash": hash(tuple(r.support.nodes.tolist()))}))
