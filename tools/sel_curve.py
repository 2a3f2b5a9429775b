"""Per-iteration t1 (group scan) and t2 (append) of a selection as functions
of the support count n: least-squares fits t1 ~ a + b n (scan of card rows x n
supports) and t2 ~ a + b n + c n^2 (append: row products over packed
triangles), per launch shape region, against the ideal rates (FP64 peak for
the scan pairs, HBM bandwidth for the triangle bytes).

    python tools/sel_curve.py [--config 3]
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--out", default=None)
args = ap.parse_args()
wl = W.config(args.config, nv=16)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=0)
P.gcb_select(b, cfg)
r = P.gcb_select(b, cfg)
rec = r.history.records
ke = np.array([x.kernel_evals for x in rec], dtype=float)
t1 = np.array([x.t1_s for x in rec]) * 1e6
t2 = np.array([x.t2_s for x in rec]) * 1e6
card = wl.nb / cfg.m
n = ke / card  # supports at the scan
out = {"config": args.config, "nc": len(r.support), "iterations": len(rec), "t1_ms": t1.sum() / 1e3,
       "t2_ms": t2.sum() / 1e3, "bins": []}
edges = [0, 384, 1024, 2048, 3072, 4096, 1 << 30]
for lo, hi in zip(edges[:-1], edges[1:]):
    sel = (n >= lo) & (n < hi) & (ke > 0)
    if sel.sum() < 8:
        continue
    a1 = np.polyfit(n[sel], t1[sel], 1)
    app = sel & (t2 > 0)
    a2 = np.polyfit(n[app], t2[app], 2) if app.sum() >= 8 else [0, 0, 0]
    out["bins"].append({"n": [lo, min(hi, int(n.max()) + 1)], "iters": int(sel.sum()), "appends": int(app.sum()),
                        "t1_us_mean": float(t1[sel].mean()), "t1_fit_a_us": float(a1[1]),
                        "t1_fit_b_ns_per_support": float(a1[0] * 1e3),
                        "t1_ideal_b_ns_per_support": float(card * 22 / 36.4e12 * 1e9),
                        "t2_us_mean": float(t2[app].mean()) if app.any() else 0.0,
                        "t2_fit": [float(x) for x in a2]})
print(json.dumps(out, indent=1))
if args.out:
    Path(args.out).write_text(json.dumps(out))
