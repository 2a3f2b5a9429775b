"""Boundary metrics on the B200 (reference metrics.py:45-115): nearest-support
distances (bit-identical to cdist), KL divergence, error summaries and
histories -- against the reference's golden vectors and the known answers
its own test-suite uses (tests/test_metrics.py of the reference)."""

import math

import numpy as np
import pytest

import rbf_oracle as O
from conftest import load_golden

pytestmark = pytest.mark.gpu


def boundary(P, pts, disp=None):
    pts = np.asarray(pts, dtype=float)
    disp = np.zeros_like(pts) if disp is None else np.asarray(disp, dtype=float)
    return P.BoundarySet(indices=np.arange(len(pts)), points=pts, disp=disp)


def support_of(P, b, rows, weights=None):
    rows = np.asarray(rows)
    w = np.zeros((len(rows), 3)) if weights is None else weights
    return P.SupportSet(nodes=b.indices[rows], points=b.points[rows], weights=w)


def empty_support(P):
    return P.SupportSet(np.empty(0, int), np.empty((0, 3)), np.empty((0, 3)))


# ------------------------------------------------------------- golden case
def golden_inputs(P):
    g = load_golden("metrics_smooth3")
    b = P.BoundarySet(indices=g["ids"], points=g["points"], disp=g["disp"])
    pos = np.searchsorted(g["ids"], g["sup_nodes"])
    rpos = np.searchsorted(g["ids"], g["rnd_nodes"])
    s = P.SupportSet(g["sup_nodes"], g["points"][pos], g["sup_weights"])
    rnd = P.SupportSet(g["rnd_nodes"], g["points"][rpos], g["rnd_weights"])
    return g, b, s, rnd


def test_nearest_distances_bitwise_golden(cuda):
    from paper_2004_04817_b200 import metrics as M

    g, b, s, rnd = golden_inputs(cuda)
    assert np.array_equal(M._nearest_distances(s, b), g["nearest"])
    assert np.array_equal(M._nearest_distances(rnd, b), g["nearest_rnd"])


def test_kl_divergence_golden(cuda):
    g, b, s, rnd = golden_inputs(cuda)
    # identical distances + the reference's numpy expression: identical bits
    assert cuda.kl_divergence(s, rnd, b) == float(g["kl"])
    assert cuda.kl_divergence(rnd, s, b) == float(g["kl_rev"])


def test_error_summary_golden(cuda):
    g, b, s, _ = golden_inputs(cuda)
    summ = cuda.error_summary(b, s, float(g["radius"]))
    assert summ.node_of_max == int(g["summary_node"])
    assert summ.max_error == pytest.approx(float(g["summary"][0]), rel=1e-9)
    assert summ.rms_error == pytest.approx(float(g["summary"][1]), rel=1e-9)


def test_error_history_golden(cuda):
    g, b, s, _ = golden_inputs(cuda)
    hist = cuda.error_history(b, s.nodes, float(g["radius"]), every=10)
    assert [n for n, _ in hist] == g["hist_n"].tolist()
    assert [h.node_of_max for _, h in hist] == g["hist_node"].tolist()
    np.testing.assert_allclose([h.max_error for _, h in hist], g["hist_max"], rtol=1e-9)
    np.testing.assert_allclose([h.rms_error for _, h in hist], g["hist_rms"], rtol=1e-9)


def test_nearest_large_matches_oracle_bitwise(cuda, rng):
    from paper_2004_04817_b200 import metrics as M

    pts = rng.normal(size=(50_000, 3))
    sp = rng.normal(size=(1_300, 3)) * 1.3
    assert np.array_equal(M._nearest_device(pts, sp), O.nearest_distances(pts, sp))


# ------------------------------------------- nearest_support_distance cases
def test_nearest_zero_for_member(cuda, rng):
    b = boundary(cuda, rng.normal(size=(8, 3)))
    assert cuda.nearest_support_distance(5, support_of(cuda, b, [2, 5]), b) == 0.0


def test_nearest_single_and_hand_cases(cuda):
    b = boundary(cuda, [[0, 0, 0], [0, 0, 2.0]])
    assert cuda.nearest_support_distance(0, support_of(cuda, b, [1]), b) == 2.0
    b = boundary(cuda, [[0, 0, 0], [1, 0, 0], [0, 3, 0], [0, 0, 7]])
    assert cuda.nearest_support_distance(0, support_of(cuda, b, [1, 2, 3]), b) == 1.0


def test_nearest_matches_brute_force_loop(cuda, rng):
    for _ in range(20):
        b = boundary(cuda, rng.normal(size=(15, 3)))
        rows = rng.choice(15, size=4, replace=False)
        s = support_of(cuda, b, rows)
        for i in range(15):
            brute = min(math.sqrt((b.points[i, 0] - p[0]) ** 2 + (b.points[i, 1] - p[1]) ** 2
                                  + (b.points[i, 2] - p[2]) ** 2) for p in s.points)
            assert cuda.nearest_support_distance(i, s, b) == pytest.approx(brute, rel=1e-15, abs=0.0)


def test_nearest_empty_support_raises(cuda, rng):
    b = boundary(cuda, rng.normal(size=(4, 3)))
    with pytest.raises(cuda.errors.EmptySupportSetError):
        cuda.nearest_support_distance(0, empty_support(cuda), b)


# ------------------------------------------------------------ KL divergence
def test_kl_identical_sets_exact_zero(cuda, rng):
    b = boundary(cuda, rng.normal(size=(20, 3)))
    s = support_of(cuda, b, [1, 7, 13])
    assert cuda.kl_divergence(s, s, b) == 0.0


def test_kl_log_two(cuda):
    b = boundary(cuda, [[0, 0, 0], [3.0, 0, 0]])
    s1 = cuda.SupportSet(np.array([0]), np.array([[1.0, 0, 0]]), np.zeros((1, 3)))
    s2 = cuda.SupportSet(np.array([0]), np.array([[2.0, 0, 0]]), np.zeros((1, 3)))
    assert cuda.kl_divergence(s1, s2, b) == pytest.approx(np.log(2.0), rel=1e-12)


def test_kl_zero_distances_and_empty(cuda, rng):
    b = boundary(cuda, rng.normal(size=(10, 3)))
    assert cuda.kl_divergence(support_of(cuda, b, np.arange(10)), support_of(cuda, b, [0]), b) == 0.0
    with pytest.raises(cuda.errors.EmptySupportSetError):
        cuda.kl_divergence(empty_support(cuda), support_of(cuda, b, [0]), b)


# ----------------------------------------------------------- error summary
def test_summary_zero_field(cuda, rng):
    b = boundary(cuda, rng.normal(size=(6, 3)))
    summ = cuda.error_summary(b, support_of(cuda, b, [0, 3]), 2.0)
    assert summ.max_error == 0.0 and summ.rms_error == 0.0


def test_summary_equal_residuals_tie_low(cuda, rng):
    b = boundary(cuda, rng.normal(size=(5, 3)), np.tile([0.0, 3.0, 4.0], (5, 1)))
    summ = cuda.error_summary(b, support_of(cuda, b, [0]), 1e-6)
    assert summ.max_error == 5.0 and summ.rms_error == pytest.approx(5.0) and summ.node_of_max == 0


def test_summary_four_hand_residuals(cuda):
    pts = np.array([[0, 0, 0], [10, 0, 0], [20, 0, 0], [30, 0, 0.0]])
    disp = np.array([[1, 0, 0], [0, 2, 0], [0, 0, 4], [2, 0, 0.0]])
    b = boundary(cuda, pts, disp)
    summ = cuda.error_summary(b, support_of(cuda, b, [0]), 1e-9)
    assert summ.max_error == 4.0 and summ.node_of_max == 2
    assert summ.rms_error == pytest.approx(np.sqrt((1 + 4 + 16 + 4) / 4))


def test_summary_rms_at_most_max_and_oracle(cuda, rng):
    pts, disp = rng.normal(size=(40, 3)), rng.normal(size=(40, 3))
    b = boundary(cuda, pts, disp)
    w = rng.normal(size=(3, 3))
    summ = cuda.error_summary(b, support_of(cuda, b, [1, 2, 3], w), 3.0)
    assert summ.rms_error <= summ.max_error
    mx, rms, node = O.error_summary(pts, disp, b.indices, pts[[1, 2, 3]], w, 3.0)
    assert summ.node_of_max == node
    assert summ.max_error == pytest.approx(mx, rel=1e-12)
    assert summ.rms_error == pytest.approx(rms, rel=1e-12)


# ----------------------------------------------------------- error history
def test_history_prefix_summaries(cuda):
    rng = np.random.default_rng(7)
    u, v = rng.uniform(0.0, 2.0 * np.pi, 200), rng.uniform(0.0, 1.0, 200)
    pts = np.column_stack([np.cos(u) * np.sqrt(1 - v**2), np.sin(u) * np.sqrt(1 - v**2), v])
    b = boundary(cuda, pts, np.tile([0.1, -0.05, 0.02], (200, 1)))
    res = cuda.greedy_select(b, cuda.SelectionConfig(radius=20.0, tol=1e-6, max_supports=200))
    hist = cuda.error_history(b, res.support.nodes, 20.0, every=10)
    counts = [n for n, _ in hist]
    assert counts[-1] == len(res.support)
    assert all(y > x for x, y in zip(counts, counts[1:]))
    assert hist[-1][1].max_error <= 1e-6
    ref = O.error_history(pts, b.disp, b.indices, res.support.nodes, 20.0, every=10)
    for (n, h), (n2, (mx, rms, node)) in zip(hist, ref):
        assert n == n2 and h.node_of_max == node
        assert h.max_error == pytest.approx(mx, rel=1e-4, abs=1e-9)
