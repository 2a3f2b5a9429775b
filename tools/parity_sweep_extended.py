"""Extended randomised parity sweep (the generator of
tests/test_gpu_parity_sweep.py over many more seeds): every launch shape of the
device selection loop against the CPU oracle; writes a JSON summary (problems,
selections compared, mismatching sequences / records, the largest weight
deviation) for profiles/.

    python tools/parity_sweep_extended.py --first 12 --count 300 --out gpurun_out/parity_sweep.json
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))
sys.path.insert(0, str(REPO / "tests"))
import paper_2004_04817_b200 as P  # noqa: E402
import rbf_oracle as O  # noqa: E402  (the checker: test infrastructure)
from paper_2004_04817_b200 import _native as N  # noqa: E402
from paper_2004_04817_b200.selection import _gcb_run  # noqa: E402
from test_gpu_parity_sweep import problem, rel  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--first", type=int, default=12)
ap.add_argument("--count", type=int, default=300)
ap.add_argument("--out", default=None)
args = ap.parse_args()
modes = {"auto": None, "msg": N.GCB_MSG, "smem": N.GCB_SMEM, "cluster": N.GCB_CLUSTER, "grid": N.GCB_GRID}
out = {"first_seed": args.first, "problems": 0, "raised": 0, "selections": 0, "supports_total": 0,
       "sequence_mismatch": [], "record_mismatch": [], "error_mismatch": [], "weights_rel_max": 0.0,
       "weights_rel_over_1e-9": []}
t0 = time.time()
for seed in range(args.first, args.first + args.count):
    pts, disp, m, radius, tol, cap = problem(seed)
    nb = len(pts)
    b = P.BoundarySet(np.arange(nb), pts, disp)
    cfg = P.SelectionConfig(radius=radius, tol=tol, max_supports=cap, m=m, seed=seed)
    out["problems"] += 1
    try:
        ref = O.select(pts, disp, radius, tol, cap, m, seed)
    except (RuntimeError, ArithmeticError) as exc:
        out["raised"] += 1
        want = P.errors.SelectionStalledError if isinstance(exc, RuntimeError) else P.errors.NotPositiveDefiniteError
        for name, mode in modes.items():
            try:
                _gcb_run(b, cfg, mode=mode)
                out["error_mismatch"].append([seed, name, "no error"])
            except want:
                pass
            except Exception as e:  # noqa: BLE001
                out["error_mismatch"].append([seed, name, type(e).__name__])
        continue
    floor = 1e-10 * float(np.linalg.norm(disp, axis=1).max())
    for name, mode in modes.items():
        try:
            res = _gcb_run(b, cfg, mode=mode)
        except Exception as e:  # noqa: BLE001
            out["error_mismatch"].append([seed, name, type(e).__name__])
            continue
        out["selections"] += 1
        out["supports_total"] += len(res.support)
        if not np.array_equal(res.support.nodes, ref["seq"]):
            out["sequence_mismatch"].append([seed, name, int(len(res.support)), int(len(ref["seq"]))])
            continue
        recs = res.history.records
        bad = len(recs) != len(ref["records"]) or any(
            (r.local_max_error > floor or q[3] > floor) and r.node != int(q[2])
            for r, q in zip(recs, ref["records"]))
        if bad:
            out["record_mismatch"].append([seed, name])
        w = rel(res.support.weights, ref["weights"])
        out["weights_rel_max"] = max(out["weights_rel_max"], w)
        if w > 1e-9:
            out["weights_rel_over_1e-9"].append([seed, name, w])
out["seconds"] = round(time.time() - t0, 1)
print(json.dumps(out, indent=1))
if args.out:
    Path(args.out).write_text(json.dumps(out, indent=1))
