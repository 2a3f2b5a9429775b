"""Small end-to-end case for compute-sanitizer (every kernel path once):
MSG selection (with a near-duplicate rejection), SMEM / CLUSTER / GRID
selections, a one-cluster selection whose closing run goes to the whole-GPU
tail launch (m = 16: run resolution + final sweep), a loop without its final
sweep (RBF_GCB_NO_SWEEP) plus the sharded-sweep kernels (error scan into a
device record, the record fold), volume evaluation, the error scan, nearest
distances, Cholesky append/solve.

    compute-sanitizer --tool {memcheck,racecheck,synccheck,initcheck} python tools/sanitize_case.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200.selection import _gcb_run  # noqa: E402

rng = np.random.default_rng(3)
pts = rng.uniform(-1, 1, (600, 3))
pts[5] = pts[9] + 1e-14  # near duplicate
disp = 0.1 * np.sin(pts @ rng.normal(size=(3, 3)))
b = P.BoundarySet(np.arange(600), pts, disp)
cfg = P.SelectionConfig(radius=2.0, tol=1e-6, max_supports=120, m=4, seed=1)
for mode in (N.GCB_MSG, N.GCB_SMEM, N.GCB_CLUSTER, N.GCB_GRID):
    res = _gcb_run(b, cfg, mode=mode)
    print(mode, len(res.support))
cfg16 = P.SelectionConfig(radius=2.0, tol=1e-5, max_supports=120, m=16, seed=2)
res16 = _gcb_run(b, cfg16)  # AUTO: MSG + tail launches
print("m16", len(res16.support))
res_ns = _gcb_run(b, cfg16, sweep=False)
import torch  # noqa: E402

lib = N.require_cuda()
pd, dd = torch.from_numpy(pts).cuda(), torch.from_numpy(disp).cuda()
sp, sw = torch.from_numpy(res_ns.support.points).cuda(), torch.from_numpy(res_ns.support.weights).cuda()
recs = torch.empty((3, 2), dtype=torch.float64, device="cuda")
for r, (lo, hi) in enumerate(((0, 250), (250, 600), (600, 600))):
    nb_ = lib.rbf_errors_scratch_bytes(max(hi - lo, 1))
    scr = torch.empty(nb_, dtype=torch.uint8, device="cuda")
    N.check(lib.rbf_errors_argmax_dev(N.dptr(pd[lo:hi]) if hi > lo else N.dptr(pd),
                                      N.dptr(dd[lo:hi]) if hi > lo else N.dptr(dd), None, hi - lo,
                                      N.dptr(sp), N.dptr(sw), sp.shape[0], 2.0, None, lo,
                                      N.dptr(recs[r]), N.dptr(scr), nb_, N.stream_ptr()), "dev")
best = torch.empty(2, dtype=torch.float64, device="cuda")
N.check(lib.rbf_best_fold(N.dptr(recs), 3, N.dptr(best), N.stream_ptr()), "fold")
print("sharded sweep", best.tolist(), res16.history.final_sweep.local_max_error)
kl = P.kl_divergence(res16.support, res.support, b)
u = P.deform_points(rng.normal(size=(5000, 3)), res.support, 2.0)
node, err = P.group_arg_max_error(b.indices[:100], b, res.support, 2.0)
st = P.CholeskyState()
a = P.assemble_phi(pts[:40], 2.0)
for k in range(40):
    st.append(a[k, : k + 1])
x = st.solve(rng.normal(size=(40, 3)))
print("ok", u.shape, node, float(err), x.shape)
