"""Generate golden vectors by running the REFERENCE package itself.

Run here (the build container, where /root/reference exists):

    python tests/golden/make_golden.py

Each case is written to tests/golden/<name>.npz. Inputs come either from
small explicit arrays (stored) or from the seeded generators in
``paper_2004_04817_b200.workloads`` (stored as parameters plus a SHA-256 of
the generated arrays, so tests can detect generator drift). Outputs are
what the reference returns: the support-node sequence, weights, the
iteration records without timing columns, the final sweep, and
displacements at a fixed sample of volume targets.

Recorded environment: numpy / scipy / OpenBLAS versions go into each file.
"""

import hashlib
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, "/root/reference/pkg/src")

import rbfdeform as R  # noqa: E402  (the reference)
from rbfdeform import core as RC  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def env():
    import scipy

    return f"numpy {np.__version__}; scipy {scipy.__version__}"


def run_selection(points, disp, radius, tol, max_supports, m, seed):
    b = R.BoundarySet(indices=np.arange(len(points)), points=points, disp=disp)
    cfg = R.SelectionConfig(radius=radius, tol=tol, max_supports=max_supports, m=m, seed=seed)
    res = R.gcb_select(b, cfg)
    recs = res.history.records
    f = res.history.final_sweep
    return {
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
        "params": np.array([radius, tol, max_supports, m, seed], dtype=float),
    }, res


def hemisphere():
    rng = np.random.default_rng(7)
    u = rng.uniform(0.0, 2.0 * np.pi, 200)
    v = rng.uniform(0.0, 1.0, 200)
    pts = np.column_stack([np.cos(u) * np.sqrt(1 - v**2), np.sin(u) * np.sqrt(1 - v**2), v])
    return pts, np.tile([0.1, -0.05, 0.02], (200, 1))


def smooth(seed):
    rng = np.random.default_rng(seed)
    nb = int(rng.integers(50, 501))
    pts = rng.uniform(-1.0, 1.0, size=(nb, 3))
    coef = rng.normal(scale=0.8, size=(3, 3))
    disp = np.stack([0.2 * np.sin(pts @ coef[i]) for i in range(3)], axis=1)
    return pts, disp


def save(name, **arrays):
    np.savez_compressed(HERE / f"{name}.npz", env=np.array(env()), **arrays)
    print("wrote", name, {k: getattr(v, "shape", None) for k, v in arrays.items()})


def volume_sample(wl, support, radius, n=4096):
    idx = np.linspace(0, wl.nv - 1, min(n, wl.nv)).astype(np.int64)
    u = R.evaluate_displacements(wl.volume[idx], support, radius)
    return idx, u


def main():
    if len(sys.argv) > 1 and sys.argv[1] in ("metrics", "meshio", "auto_m"):  # from this case on
        return metrics_only()
    # 1. explicit small inputs (stored)
    pts, disp = hemisphere()
    for m in (1, 4):
        out, _ = run_selection(pts, disp, 5.0, 1e-6, 100, m, 5)
        save(f"hemisphere_m{m}", points=pts, disp=disp, **out)
    for seed in (0, 3, 11):
        pts, disp = smooth(seed)
        for m in (1, 5):
            out, _ = run_selection(pts, disp, 3.0, 1e-4, min(len(pts), 80), m, seed)
            save(f"smooth{seed}_m{m}", points=pts, disp=disp, **out)

    # a run long enough (n = 1200) to cross the shared-memory path's capacity
    rng = np.random.default_rng(77)
    pts = rng.uniform(0, 1, (4000, 3))
    disp = np.stack([0.05 * np.sin(4 * pts[:, 0] + 1), 0.05 * np.cos(3 * pts[:, 1]),
                     0.05 * np.sin(5 * pts[:, 2] + pts[:, 0])], 1)
    out, _ = run_selection(pts, disp, 0.25, 1e-7, 1200, 8, 3)
    save("switch_m8", points=pts, disp=disp, **out)

    # 2. evaluation and factor known answers
    rng = np.random.default_rng(1234)
    sp = rng.normal(size=(700, 3))
    sw = rng.normal(size=(700, 3))
    q = rng.normal(size=(5000, 3)) * 2.0
    s = R.SupportSet(nodes=np.arange(700), points=sp, weights=sw)
    save("eval_random", sup_points=sp, sup_weights=sw, targets=q,
         u=R.evaluate_displacements(q, s, 1.5), radius=np.array(1.5))
    a_pts = rng.normal(size=(150, 3))
    a = R.assemble_phi(a_pts, 3.0)
    st = R.CholeskyState()
    for k in range(150):
        st.append(a[k, : k + 1])
    rhs = rng.normal(size=(150, 3))
    save("chol150", points=a_pts, L=st.factor, rhs=rhs, x=st.solve(rhs), radius=np.array(3.0))

    # 2b. metrics (reference metrics.py): nearest distances, KL, summaries, history
    from rbfdeform import metrics as RM

    pts, disp = smooth(3)
    b = R.BoundarySet(indices=np.arange(len(pts)) * 3 + 1, points=pts, disp=disp)
    res = R.gcb_select(b, R.SelectionConfig(radius=3.0, tol=1e-4, max_supports=60, m=4, seed=2))
    rnd = R.random_select(b, 25, seed=9, radius=3.0)
    summ = RM.error_summary(b, res.support, 3.0)
    hist = RM.error_history(b, res.support.nodes, 3.0, every=10)
    save("metrics_smooth3", points=pts, disp=disp, ids=b.indices, sup_nodes=res.support.nodes,
         sup_weights=res.support.weights, rnd_nodes=rnd.nodes, rnd_weights=rnd.weights,
         nearest=RM._nearest_distances(res.support, b), nearest_rnd=RM._nearest_distances(rnd, b),
         kl=np.array(RM.kl_divergence(res.support, rnd, b)),
         kl_rev=np.array(RM.kl_divergence(rnd, res.support, b)),
         summary=np.array([summ.max_error, summ.rms_error]), summary_node=np.array(summ.node_of_max),
         hist_n=np.array([n for n, _ in hist]), hist_max=np.array([h.max_error for _, h in hist]),
         hist_rms=np.array([h.rms_error for _, h in hist]),
         hist_node=np.array([h.node_of_max for _, h in hist]), radius=np.array(3.0))

    # 2c. meshio (reference meshio.py): canonical writer output, for byte parity
    from rbfdeform import meshio as RIO

    rng = np.random.default_rng(99)
    nodes = rng.normal(size=(40, 3)) * np.array([1.0, 1e-7, 3e5])
    nodes[0] = [0.0, -0.0, 1e-310]
    nodes[1] = [1.0, 0.1, 123456789.0]
    mesh = RIO.Mesh(nodes=nodes, boundary=np.array([5, 1, 30, 2]),
                    cells=[np.array([0, 1, 2]), np.array([3, 4, 5, 6])])
    disp = rng.normal(size=(4, 3)) * 1e-3
    res = R.gcb_select(R.BoundarySet(np.arange(40), nodes[:, :3] * np.array([1.0, 1e7, 3e-6]),
                                     rng.normal(size=(40, 3)) * 0.01),
                       R.SelectionConfig(radius=3.0, tol=1e-6, max_supports=12, m=3, seed=1))
    (HERE / "meshio_mesh.mdk1").write_text(RIO.write_mesh(mesh))
    (HERE / "meshio_disp.mdk1").write_text(RIO.write_displacements(disp, mesh.boundary))
    (HERE / "meshio_history.csv").write_text(RIO.write_history_csv(res.history))
    (HERE / "meshio_supports.csv").write_text(RIO.write_supports_csv(res.support))
    save("meshio_values", nodes=nodes, boundary=mesh.boundary, disp=disp,
         sup_nodes=res.support.nodes, sup_points=res.support.points, sup_weights=res.support.weights)

    # 2d. resolve_auto_m (reference cli.py:69-99) on configs[0]'s wing
    from rbfdeform.cli import resolve_auto_m

    wl0 = W.config(0, nv=10)
    b0 = R.BoundarySet(indices=np.arange(wl0.nb), points=wl0.points, disp=wl0.disp)
    cases = [(200, wl0.tol), (40, wl0.tol), (200, 1e-2)]
    save("auto_m", caps=np.array([c for c, _ in cases]), tols=np.array([t for _, t in cases]),
         m=np.array([resolve_auto_m(b0, wl0.radius, t, seed=0, probe_cap=c) for c, t in cases]),
         digest=np.array(digest(wl0.points, wl0.disp)))

    # 3. BASELINE configs (generator parameters + digest; outputs)
    for idx, ms in ((0, (1, 8)),):
        wl = W.config(idx, nv=100_000)
        for m in ms:
            out, res = run_selection(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, m, 0)
            vidx, u = volume_sample(wl, res.support, wl.radius)
            save(f"cfg{idx}_m{m}", digest=np.array(digest(wl.points, wl.disp, wl.volume)),
                 vol_idx=vidx, vol_u=u, **out)
    wl = W.config(1, nv=2_000_000)
    out, res = run_selection(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 32, 0)
    vidx, u = volume_sample(wl, res.support, wl.radius)
    save("cfg1_m32", digest=np.array(digest(wl.points, wl.disp, wl.volume)), vol_idx=vidx, vol_u=u, **out)
    wl = W.config(2, nv=200_000)  # BASELINE configs[2] at full boundary size
    out, res = run_selection(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 48, 0)
    vidx, u = volume_sample(wl, res.support, wl.radius)
    save("cfg2_m48", digest=np.array(digest(wl.points, wl.disp)), vol_idx=vidx, vol_u=u, **out)
    # BASELINE configs[3] at full boundary size (Nb = 200k, m = 64, R = 4), first 400 supports
    wl = W.config(3, nv=100_000)
    out, res = run_selection(wl.points, wl.disp, wl.radius, wl.tol, 400, 64, 0)
    vidx, u = volume_sample(wl, res.support, wl.radius)
    save("cfg3_m64_cap400", digest=np.array(digest(wl.points, wl.disp)), vol_idx=vidx, vol_u=u, **out)
    wl = W.structured_wing(n_span=60, n_section=200, nv=100_000, m=48, name="cfg2s")
    out, res = run_selection(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 48, 0)
    vidx, u = volume_sample(wl, res.support, wl.radius)
    save("cfg2s_m48", digest=np.array(digest(wl.points, wl.disp, wl.volume)), vol_idx=vidx, vol_u=u, **out)


def metrics_only():
    src = open(__file__).read()
    start = {"metrics": "    # 2b. metrics", "meshio": "    # 2c. meshio", "auto_m": "    # 2d. resolve_auto_m"}
    a = src.index(start[sys.argv[1]])
    b = src.index("    # 3. BASELINE configs")
    exec(compile("if True:\n" + src[a:b], __file__, "exec"), globals())


if __name__ == "__main__":
    main()
