"""Pin the CPU oracle (oracle/rbf_oracle.py) against golden vectors that
tests/golden/make_golden.py produced by running the reference itself, and
directly against the reference when it is importable (build container)."""

import numpy as np
import pytest

import rbf_oracle as O
from conftest import import_reference, load_golden, reference_available
from paper_2004_04817_b200 import workloads as W

SELECTION_CASES = [
    "hemisphere_m1", "hemisphere_m4", "smooth0_m1", "smooth0_m5", "smooth3_m1",
    "smooth3_m5", "smooth11_m1", "smooth11_m5", "cfg0_m1", "cfg0_m8", "switch_m8",
    "cfg2_m48", "cfg3_m64_cap400",
]


def inputs_for(name, g):
    if "points" in g:
        return g["points"], g["disp"], None
    if name.startswith("cfg0"):
        wl = W.config(0, nv=100_000)
    elif name.startswith("cfg1"):
        wl = W.config(1, nv=2_000_000)
    elif name == "cfg2_m48":
        wl = W.config(2, nv=200_000)
    elif name.startswith("cfg3"):
        wl = W.config(3, nv=100_000)
    else:
        wl = W.structured_wing(n_span=60, n_section=200, nv=100_000, m=48, name="cfg2s")
    return wl.points, wl.disp, wl


def check_selection(out, g):
    assert np.array_equal(out["seq"], g["seq"])
    assert np.array_equal(out["weights"], g["weights"])
    recs = out["records"]
    assert [r[0] for r in recs] == g["rec_iter"].tolist()
    assert [r[1] for r in recs] == g["rec_group"].tolist()
    assert [r[2] for r in recs] == g["rec_node"].tolist()
    assert np.array_equal(np.array([r[3] for r in recs]), g["rec_local_max"])
    assert [r[4] for r in recs] == g["rec_evals"].tolist()
    f = out["final"]
    assert [f[0], f[1], f[3]] == [g["final"][0], g["final"][1], g["final"][2]]
    assert f[2] == g["final_max"]
    assert out["converged"] == bool(g["converged"])


@pytest.mark.parametrize("name", SELECTION_CASES)
def test_oracle_selection_matches_reference_golden(name):
    g = load_golden(name)
    pts, disp, wl = inputs_for(name, g)
    radius, tol, cap, m, seed = g["params"]
    out = O.select(pts, disp, radius, tol, int(cap), int(m), int(seed))
    check_selection(out, g)
    if wl is not None:
        u = O.eval_sum(wl.volume[g["vol_idx"]], pts[out["seq"]], out["weights"], radius)
        assert np.array_equal(u, g["vol_u"])


def test_generator_digests_stable():
    import hashlib

    for name, wl in (("cfg0_m8", W.config(0, nv=100_000)),):
        h = hashlib.sha256()
        for a in (wl.points, wl.disp, wl.volume):
            h.update(np.ascontiguousarray(a).tobytes())
        assert h.hexdigest() == str(load_golden(name)["digest"])


def test_oracle_eval_matches_golden():
    g = load_golden("eval_random")
    u = O.eval_sum(g["targets"], g["sup_points"], g["sup_weights"], float(g["radius"]))
    assert np.array_equal(u, g["u"])


def test_oracle_eval_threads_bitwise():
    g = load_golden("eval_random")
    a = O.eval_sum(g["targets"], g["sup_points"], g["sup_weights"], 1.5, threads=1)
    b = O.eval_sum(g["targets"], g["sup_points"], g["sup_weights"], 1.5, threads=4)
    assert np.array_equal(a, b)


def test_oracle_factor_matches_golden():
    g = load_golden("chol150")
    pts = g["points"]
    f = O.Factor()
    for k in range(len(pts)):
        d = np.sqrt(((pts[k] - pts[: k + 1]) ** 2).sum(1))
        from scipy.spatial.distance import cdist

        row = O.phi(cdist(pts[k : k + 1], pts[: k + 1])[0] / float(g["radius"]))
        row[k] = 1.0
        assert f.try_append(row) > 0
    assert np.array_equal(f.L, g["L"])
    assert np.array_equal(f.solve(g["rhs"]), g["x"])


def test_oracle_known_answers():
    assert O.phi(np.array(0.5)) == pytest.approx(0.1875, abs=1e-15)
    assert O.phi(np.array(0.0)) == 1.0 and O.phi(np.array(1.0)) == 0.0
    assert O.argmax_low(np.array([1.0, 3.0, 3.0]), np.array([5, 9, 2])) == 2
    # golden PCG64 triple of the reference tests (test_selection.py:310-314)
    assert np.random.default_rng(2024).choice(10, size=3, replace=False).tolist() == [6, 0, 1]


def test_oracle_stall_and_notpd():
    # two coincident nodes with opposite displacements (the construction of
    # reference tests/test_selection.py:262-272)
    pts = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 0]])
    disp = np.zeros((4, 3))
    disp[0] = [1.0, 0, 0]
    disp[3] = [-1.0, 0, 0]
    with pytest.raises(RuntimeError):
        O.select(pts, disp, 3.0, 1e-9, 4, 1, 0)
    same = np.zeros((4, 3))
    with pytest.raises(ArithmeticError):
        O.select(same, np.ones((4, 3)), 2.0, 1e-6, 4, 1, 0)


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
@pytest.mark.parametrize("seed", [21, 22])
def test_oracle_matches_reference_live(seed):
    R = import_reference()
    rng = np.random.default_rng(seed)
    nb = int(rng.integers(200, 600))
    pts = rng.uniform(-1, 1, (nb, 3))
    disp = 0.1 * np.sin(pts @ rng.normal(size=(3, 3)))
    for m in (1, 3):
        b = R.BoundarySet(np.arange(nb), pts, disp)
        ref = R.gcb_select(b, R.SelectionConfig(radius=2.5, tol=1e-5, max_supports=nb, m=m, seed=seed))
        out = O.select(pts, disp, 2.5, 1e-5, nb, m, seed)
        assert np.array_equal(out["seq"], ref.support.nodes)
        assert np.array_equal(out["weights"], ref.support.weights)
        q = rng.normal(size=(3000, 3))
        assert np.array_equal(O.eval_sum(q, ref.support.points, ref.support.weights, 2.5),
                              R.evaluate_displacements(q, ref.support, 2.5))


def test_oracle_metrics_match_reference_golden():
    """nearest distances, KL, error summary and history (reference metrics.py)
    restated in the oracle reproduce the reference's bits."""
    g = load_golden("metrics_smooth3")
    pts, disp, ids, r = g["points"], g["disp"], g["ids"], float(g["radius"])
    pos = np.searchsorted(ids, g["sup_nodes"])
    rpos = np.searchsorted(ids, g["rnd_nodes"])
    assert np.array_equal(O.nearest_distances(pts, pts[pos]), g["nearest"])
    assert np.array_equal(O.nearest_distances(pts, pts[rpos]), g["nearest_rnd"])
    assert O.kl_divergence(pts, pts[pos], pts[rpos]) == float(g["kl"])
    assert O.kl_divergence(pts, pts[rpos], pts[pos]) == float(g["kl_rev"])
    mx, rms, node = O.error_summary(pts, disp, ids, pts[pos], g["sup_weights"], r)
    assert (mx, rms) == tuple(g["summary"].tolist()) and node == int(g["summary_node"])
    hist = O.error_history(pts, disp, ids, g["sup_nodes"], r, every=10)
    assert [n for n, _ in hist] == g["hist_n"].tolist()
    assert [h[0] for _, h in hist] == g["hist_max"].tolist()
    assert [h[1] for _, h in hist] == g["hist_rms"].tolist()
    assert [h[2] for _, h in hist] == g["hist_node"].tolist()


@pytest.mark.parametrize("name", ["cfg3_m64", "cfg4_m1", "cfg4_m94", "cfg4_m141", "cfg4_m187", "cfg4_stress"])
def test_large_goldens_match_generator(name):
    """The large reference runs (tests/golden/make_golden_large.py) were made on
    the current workload generators: same boundary bits, and the recorded
    second-solve spread is present."""
    from conftest import digest

    g = load_golden(name)
    wl = W.config(3, nv=10) if name.startswith("cfg3") else W.config(2, nv=10)
    assert digest(wl.points, wl.disp) == str(g["digest"])
    assert float(g["alt_u_rel"]) < 1e-7 and len(g["seq"]) == len(g["weights"])
    assert int(g["params"][2]) == (1500 if name == "cfg4_stress" else wl.nb)
