"""BASELINE.json configs[4]: group-count sweep on the config-2 geometry.

Mirrors the reference's ``cmd_bench`` (cli.py:240-281): a warm-up run of the
first m is excluded, then per m one ``gcb_select`` and one ``deform_points``
over all volume nodes, reported in the reference's row schema
(``cli.py:38``: m,n_supports,converged,iterations,cum_kernel_evals,t1_s,t2_s,t3_s)
plus device-side times. The m list is the survey's:
m = 1 (original greedy) gives Nc, then m in {Nb/Nc, 1.5 Nb/Nc, 2 Nb/Nc}.

Global-support stress: R = the bounding-box diagonal of boundary and volume
(every pair active; the volume kernel never culls, so its time is the dense
cost at any R). The selection at that R is run with a support cap and its
outcome (converged / NotPD / stalled) is reported as is.

    python tools/msweep.py [--nv 10000000] [--out gpurun_out/msweep.json]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nv", type=int, default=10_000_000)
    ap.add_argument("--stress-cap", type=int, default=1500)
    ap.add_argument("--out", default="gpurun_out/msweep.json")
    args = ap.parse_args()

    import torch

    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import _native as N
    from paper_2004_04817_b200 import workloads as W

    N.require_cuda()
    wl = W.config(2, nv=args.nv)
    boundary = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
    vol_d = torch.from_numpy(wl.volume).cuda()
    out_d = torch.empty_like(vol_d)

    def select(m, radius=wl.radius, cap=wl.nb):
        cfg = P.SelectionConfig(radius=radius, tol=wl.tol, max_supports=cap, m=m, seed=0)
        torch.cuda.synchronize()
        with N.launch_log(timing=True) as log:
            t0 = time.perf_counter()
            res = P.gcb_select(boundary, cfg)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
        dev = sum(log.kernel_ms("rbf_gcb_run")) * 1e-3
        return res, wall, dev

    def volume(res, radius=wl.radius):
        sp = torch.from_numpy(res.support.points).cuda()
        sw = torch.from_numpy(res.support.weights).cuda()
        P.eval_device(vol_d, sp, sw, radius, deform=True, out=out_d)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        P.eval_device(vol_d, sp, sw, radius, deform=True, out=out_d)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def row(m, res, wall, dev, t3):
        h = res.history
        return {
            "m": m, "n_supports": len(res.support), "converged": bool(res.converged),
            "iterations": len(h.records), "cum_kernel_evals": int(P.error_stage_cost(h)),
            "t1_s": float(sum(r.t1_s for r in h.records)), "t2_s": float(sum(r.t2_s for r in h.records)),
            "t3_s": t3, "selection_wall_s": wall, "selection_device_s": dev,
            "device_mode": getattr(h, "device_mode", None),
            "pairs_per_s_selection": int(P.error_stage_cost(h)) / dev if dev else None,
            "pairs_per_s_volume": wl.nv * len(res.support) / t3,
        }

    rows = []
    select(1)  # warm-up (cli.py:263)
    res, wall, dev = select(1)
    nc = len(res.support)
    rows.append(row(1, res, wall, dev, volume(res)))
    print(json.dumps(rows[-1]), flush=True)
    ms = [int(round(f * wl.nb / nc)) for f in (1.0, 1.5, 2.0)]
    for m in ms:
        res, wall, dev = select(m)
        rows.append(row(m, res, wall, dev, volume(res)))
        print(json.dumps(rows[-1]), flush=True)

    # global-support stress
    allp = np.vstack([wl.points, wl.volume[:: max(1, wl.nv // 1_000_000)]])
    diag = float(np.linalg.norm(allp.max(0) - allp.min(0)))
    stress = {"radius": diag, "m": ms[1], "cap": args.stress_cap}
    try:
        res, wall, dev = select(ms[1], radius=diag, cap=args.stress_cap)
        stress.update(row(ms[1], res, wall, dev, volume(res, diag)))
        stress["outcome"] = "converged" if res.converged else "cap reached"
    except Exception as exc:  # NotPD / stall are legitimate outcomes at global support
        stress["outcome"] = f"{type(exc).__name__}: {exc}"
        # dense cost at global support: the last config-4 support set evaluated at R = diag
        stress["t3_s_dense_at_diag"] = volume(res, diag)
    print(json.dumps({"stress": stress}), flush=True)

    header = "m,n_supports,converged,iterations,cum_kernel_evals,t1_s,t2_s,t3_s"
    csv = [header] + [
        f"{r['m']},{r['n_supports']},{str(r['converged']).lower()},{r['iterations']},"
        f"{r['cum_kernel_evals']},{r['t1_s']!r},{r['t2_s']!r},{r['t3_s']!r}" for r in rows
    ]
    out = {"workload": f"configs[4] on configs[2] geometry: Nb={wl.nb}, Nv={wl.nv}, R={wl.radius}, "
                       f"tol=1e-5*max|d|", "gpu": torch.cuda.get_device_name(),
           "rows": rows, "stress": stress, "csv": "\n".join(csv)}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(out, indent=1))
    print("\n".join(csv))


if __name__ == "__main__":
    main()
