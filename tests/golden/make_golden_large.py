"""Golden vectors for the LARGE BASELINE runs, produced by running the REFERENCE itself.

Companion to make_golden.py (same output schema, same ``run_selection``):

* ``cfg3_m64``        configs[3] at full size: Nb = 200k, R = 4, m = 64, every support
                      (max_supports = Nb) -- the run the survey flagged for
                      inverse-factor parity at kappa >= 1e10.
* ``cfg4_m1``         configs[4]: the original greedy (m = 1) on the configs[2] wing.
* ``cfg4_m<k>``       configs[4]: m = round(f * Nb / Nc), f in {1, 1.5, 2}, Nc from cfg4_m1.
* ``bign_m``          more than 8,192 supports (past the round-1 device limit): 9,000
                      random nodes in the unit cube, R = 0.15 (well conditioned),
                      m = Nb (single-node groups: every visit appends), cap 8,500 --
                      the loop runs MSG -> SMEM -> GRID and crosses n = 8,192.
* ``cfg4_stress``     configs[4] global-support stress: R = bounding-box diagonal of the
                      boundary and (a strided 1M sample of) the volume, m = the 1.5 Nb/Nc
                      entry, support cap 1500 (tools/msweep.py's stress).

Each file also records the reference's OWN numerical spread at that conditioning: the
weights of the same support set solved a second, equally backward-stable way (one
blocked LAPACK Cholesky of the assembled Phi, ``np.linalg.cholesky`` + two triangular
solves) and the volume displacements those weights give. ``alt_w_rel`` /
``alt_u_rel`` = max-abs deviation / max-abs value between the two; the GPU's parity bar
for a case is never looser than a small multiple of that spread (tests/test_gpu_parity.py).

The reference runs with ``workers = len(os.sched_getaffinity(0))``; its results do not
depend on ``workers`` (reference SPEC.md:254).

    python tests/golden/make_golden_large.py cfg4 cfg3     # tens of CPU minutes
"""

import os
import sys
import time

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as MG  # noqa: E402  (puts the reference and the repo on sys.path)

R, RC, W = MG.R, MG.RC, MG.W
WORKERS = len(os.sched_getaffinity(0))


def run(points, disp, radius, tol, cap, m, seed=0):
    b = R.BoundarySet(indices=np.arange(len(points)), points=points, disp=disp)
    cfg = R.SelectionConfig(radius=radius, tol=tol, max_supports=cap, m=m, seed=seed, workers=WORKERS)
    t0 = time.perf_counter()
    res = R.gcb_select(b, cfg)
    dt = time.perf_counter() - t0
    recs = res.history.records
    f = res.history.final_sweep
    out = {
        "seq": np.asarray(res.support.nodes, dtype=np.int64),
        "weights": res.support.weights,
        "rec_iter": np.array([r.iteration for r in recs], dtype=np.int64),
        "rec_group": np.array([r.group for r in recs], dtype=np.int64),
        "rec_node": np.array([r.node for r in recs], dtype=np.int64),
        "rec_local_max": np.array([r.local_max_error for r in recs], dtype=float),
        "rec_evals": np.array([r.kernel_evals for r in recs], dtype=np.int64),
        "rec_cum": np.array([r.cum_kernel_evals for r in recs], dtype=np.int64),
        "final": np.array([f.iteration, f.node, f.kernel_evals, f.cum_kernel_evals], dtype=np.int64),
        "final_max": np.array(f.local_max_error),
        "converged": np.array(res.converged),
        "params": np.array([radius, tol, cap, m, seed], dtype=float),
        "ref_select_s": np.array(dt),
        "ref_t1_s": np.array(sum(r.t1_s for r in recs)),
        "ref_t2_s": np.array(sum(r.t2_s for r in recs)),
        "workers": np.array(WORKERS),
    }
    print(f"  select m={m} R={radius:.4g}: Nc={len(res.support)} iters={len(recs)} "
          f"converged={res.converged} {dt:.1f} s", flush=True)
    return out, res


def alt_solve(points, disp, res, radius, vol_sample):
    nodes = np.asarray(res.support.nodes)
    phi = R.assemble_phi(points[nodes], radius)
    L = np.linalg.cholesky(phi)
    y = sla.solve_triangular(L, disp[nodes], lower=True)
    w_alt = sla.solve_triangular(L.T, y, lower=False)
    s_alt = R.SupportSet(nodes=nodes, points=points[nodes], weights=w_alt)
    u_ref = R.evaluate_displacements(vol_sample, res.support, radius, workers=WORKERS)
    u_alt = R.evaluate_displacements(vol_sample, s_alt, radius, workers=WORKERS)

    def rel(a, b):
        return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

    d = np.linalg.eigvalsh(phi) if len(nodes) <= 2500 else None
    out = {"alt_weights": w_alt, "alt_w_rel": np.array(rel(w_alt, res.support.weights)),
           "alt_u_rel": np.array(rel(u_alt, u_ref)),
           "kappa": np.array(float(d[-1] / d[0]) if d is not None else np.nan),
           "w_absmax": np.array(float(np.abs(res.support.weights).max()))}
    print(f"  spread: weights {out['alt_w_rel']:.3g}, displacements {out['alt_u_rel']:.3g}, "
          f"kappa {out['kappa']:.3g}, |w|max {out['w_absmax']:.3g}", flush=True)
    return out, u_ref


def vol_idx(nv, n=4096):
    return np.linspace(0, nv - 1, min(n, nv)).astype(np.int64)


def case_cfg3():
    wl = W.config(3, nv=100_000)
    out, res = run(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 64)
    idx = vol_idx(wl.nv)
    sp, u = alt_solve(wl.points, wl.disp, res, wl.radius, wl.volume[idx])
    MG.save("cfg3_m64", digest=np.array(MG.digest(wl.points, wl.disp)), vol_idx=idx, vol_u=u, **out, **sp)


def case_cfg4():
    wl = W.config(2, nv=200_000)
    dig = np.array(MG.digest(wl.points, wl.disp))
    idx = vol_idx(wl.nv)
    out, res = run(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 1)
    sp, u = alt_solve(wl.points, wl.disp, res, wl.radius, wl.volume[idx])
    MG.save("cfg4_m1", digest=dig, vol_idx=idx, vol_u=u, **out, **sp)
    nc = len(res.support)
    ms = [int(round(f * wl.nb / nc)) for f in (1.0, 1.5, 2.0)]
    for m in ms:
        out, res = run(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, m)
        sp, u = alt_solve(wl.points, wl.disp, res, wl.radius, wl.volume[idx])
        MG.save(f"cfg4_m{m}", digest=dig, vol_idx=idx, vol_u=u, **out, **sp)
    # global-support stress: R = bounding-box diagonal over the boundary and the full
    # configs[2] volume (Nv = 10M, strided to 1M points), as tools/msweep.py computes it
    wl10 = W.config(2)
    allp = np.vstack([wl10.points, wl10.volume[:: max(1, wl10.nv // 1_000_000)]])
    diag = float(np.linalg.norm(allp.max(0) - allp.min(0)))
    del wl10, allp
    try:
        out, res = run(wl.points, wl.disp, diag, wl.tol, 1500, ms[1])
    except Exception as exc:  # NotPD / stall are legitimate outcomes at global support
        print("  stress raised", type(exc).__name__, exc, flush=True)
        MG.save("cfg4_stress", digest=dig, params=np.array([diag, wl.tol, 1500, ms[1], 0], dtype=float),
                raised=np.array(type(exc).__name__), message=np.array(str(exc)))
        return
    sp, u = alt_solve(wl.points, wl.disp, res, diag, wl.volume[idx])
    MG.save("cfg4_stress", digest=dig, vol_idx=idx, vol_u=u, **out, **sp)


def case_bign():
    rng = np.random.default_rng(8192)
    pts = rng.uniform(0.0, 1.0, (9000, 3))
    disp = np.stack([0.02 * np.sin(3 * pts[:, 0] + 1), 0.02 * np.cos(2 * pts[:, 1]),
                     0.02 * np.sin(4 * pts[:, 2] + pts[:, 0])], 1)
    out, res = run(pts, disp, 0.15, 1e-300, 8500, len(pts))
    q = rng.uniform(0.0, 1.0, (4096, 3))
    u = R.evaluate_displacements(q, res.support, 0.15, workers=WORKERS)
    MG.save("bign_m", points=pts, disp=disp, targets=q, vol_u=u, **out)


if __name__ == "__main__":
    for name in sys.argv[1:] or ["cfg4", "cfg3"]:
        print("case", name, flush=True)
        globals()[f"case_{name}"]()
