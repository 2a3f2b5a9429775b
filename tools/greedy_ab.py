"""A/B helper: one warm gcb_select per m on the configs[2] boundary (Nb = 80k);
prints device time, t1/t2 sums, the device phase split and a sequence hash."""
import os, sys, time, json, numpy as np, torch
os.environ.setdefault("RBF_GCB_PHASES", "1")  # phase split (the clock costs ~4 % of the loop)
sys.path.insert(0, ".")
import paper_2004_04817_b200 as P
from paper_2004_04817_b200 import _native as N, workloads as W
wl = W.config(2, nv=1000)
b = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
for m in [int(x) for x in sys.argv[1].split(",")]:
    cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=m, seed=0)
    P.gcb_select(b, cfg)
    with N.launch_log(timing=True) as log:
        r = P.gcb_select(b, cfg); torch.cuda.synchronize()
    dev = sum(log.kernel_ms("rbf_gcb_run"))
    h = r.history
    print(json.dumps({"mode": os.environ.get("RBF_GCB_MODE"), "m": m, "nc": len(r.support), "dev_ms": dev,
          "t1_ms": 1e3*sum(x.t1_s for x in h.records), "t2_ms": 1e3*sum(x.t2_s for x in h.records), "phases_us": {k: round(v / 1.965e3, 1) for k, v in getattr(h, "device_phase_cycles", {}).items() if k.startswith("scan") or k in ("c0", "r", "c", "pivot_cols", "fold_row", "bookkeeping")}, "seq_hash": hash(tuple(r.support.nodes.tolist()))}))
