"""Time a whole-boundary error sweep (Nb rows x Nc supports + arg-max) through
the standalone fused error kernel (rbf_errors_argmax: eval_kernel<error> +
best reduction) on configs[1], for comparison with the selection's whole-GPU
tail launch that runs the same sweep inside gcb_grid_kernel (launch list).

    python tools/sweep_compare.py [--config 1]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

cfgi = int(sys.argv[sys.argv.index("--config") + 1]) if "--config" in sys.argv else 1
wl = W.config(cfgi)
cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
res = P.gcb_select(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp), cfg)
lib = N.require_cuda()
pts = torch.from_numpy(wl.points).cuda()
disp = torch.from_numpy(wl.disp).cuda()
pos = torch.arange(wl.nb, dtype=torch.int64, device="cuda")
sp = torch.from_numpy(res.support.points).cuda()
w = torch.from_numpy(res.support.weights).cuda()
nbytes = lib.rbf_errors_scratch_bytes(wl.nb)
scratch = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
best = (N.ctypes.c_double * 2)()


def sweep():
    rc = lib.rbf_errors_argmax(N.dptr(pts), N.dptr(disp), N.dptr(pos), wl.nb, N.dptr(sp), N.dptr(w),
                               sp.shape[0], float(wl.radius), None, best, N.dptr(scratch), nbytes,
                               N.stream_ptr())
    N.check(rc, "rbf_errors_argmax")


for _ in range(5):
    sweep()
torch.cuda.synchronize()
ts = []
for _ in range(20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sweep()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) * 1e3)
fin = res.history.final_sweep
print({"config": cfgi, "nb": wl.nb, "nc": int(sp.shape[0]), "sweep_us_median": float(np.median(ts)),
       "sweep_us_min": float(min(ts)), "max_err": best[0], "pos": int(best[1]),
       "loop_final_max": fin.local_max_error, "loop_final_node": int(fin.node),
       "loop_final_t1_us": fin.t1_s * 1e6})
