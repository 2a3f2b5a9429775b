"""Small end-to-end case for compute-sanitizer (every kernel path once):
MSG selection (with a near-duplicate rejection), SMEM / CLUSTER / GRID
selections, volume evaluation, error scan, Cholesky append/solve."""
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
u = P.deform_points(rng.normal(size=(5000, 3)), res.support, 2.0)
node, err = P.group_arg_max_error(b.indices[:100], b, res.support, 2.0)
st = P.CholeskyState()
a = P.assemble_phi(pts[:40], 2.0)
for k in range(40):
    st.append(a[k, : k + 1])
x = st.solve(rng.normal(size=(40, 3)))
print("ok", u.shape, node, float(err), x.shape)
