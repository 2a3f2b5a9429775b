"""Host-side logic that must match the reference exactly, and the
no-CPU-fallback contract (runs on CPU)."""

import numpy as np
import pytest

import rbf_oracle as O
import paper_2004_04817_b200 as P
from paper_2004_04817_b200 import errors as E
from paper_2004_04817_b200.selection import _partition_positions
from conftest import has_cuda, import_reference, reference_available


@pytest.mark.parametrize("nb,m,seed", [(10, 3, 0), (200, 1, 5), (20000, 32, 0), (101, 4, 7), (7, 7, 1)])
def test_partition_positions_match_oracle(nb, m, seed):
    _, flat, off = _partition_positions(nb, m, seed)
    groups = O.partition(nb, m, seed)
    assert off[-1] == nb and len(off) == m + 1
    for j in range(m):
        assert np.array_equal(flat[off[j]:off[j + 1]], groups[j])


def test_partition_boundary_api():
    b = P.BoundarySet(np.arange(0, 20, 2), np.random.default_rng(0).normal(size=(10, 3)), np.zeros((10, 3)))
    part = P.partition_boundary(b, 3, seed=4)
    assert part.m == 3 and sorted(np.concatenate(part.groups).tolist()) == b.indices.tolist()
    assert max(map(len, part.groups)) - min(map(len, part.groups)) <= 1
    with pytest.raises(E.InvalidGroupCountError):
        P.partition_boundary(b, 11, 0)
    with pytest.raises(E.InvalidGroupCountError):
        P.partition_boundary(b, 0, 0)


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_partition_and_seeds_match_reference_live():
    R = import_reference()
    rng = np.random.default_rng(3)
    pts = rng.normal(size=(500, 3))
    disp = rng.normal(size=(500, 3))
    ids = np.cumsum(rng.integers(1, 4, 500))
    rb = R.BoundarySet(ids, pts, disp)
    b = P.BoundarySet(ids, pts, disp)
    for m in (1, 6, 500):
        a = R.partition_boundary(rb, m, 9)
        c = P.partition_boundary(b, m, 9)
        assert all(np.array_equal(x, y) for x, y in zip(a.groups, c.groups))
    assert np.array_equal(R.seed_supports(rb), P.seed_supports(b))


def test_seed_norms_are_numpy_bits():
    # the device seeds use sqrt((x0*x0 + x1*x1) + x2*x2): numpy's bits for (n, 3) rows
    rng = np.random.default_rng(11)
    x = rng.normal(size=(5000, 3)) * 1e3
    assert np.array_equal(np.linalg.norm(x, axis=1), np.sqrt((x[:, 0] * x[:, 0] + x[:, 1] * x[:, 1]) + x[:, 2] * x[:, 2]))


def test_config_and_boundary_validation():
    with pytest.raises(ValueError):
        P.SelectionConfig(radius=0.0, tol=1e-6, max_supports=10)
    with pytest.raises(ValueError):
        P.SelectionConfig(radius=1.0, tol=0.0, max_supports=10)
    with pytest.raises(ValueError):
        P.SelectionConfig(radius=1.0, tol=1e-6, max_supports=2)
    with pytest.raises(E.InvalidGroupCountError):
        P.SelectionConfig(radius=1.0, tol=1e-6, max_supports=10, m=0)
    with pytest.raises(ValueError):
        P.BoundarySet(np.array([1, 1]), np.zeros((2, 3)), np.zeros((2, 3)))
    with pytest.raises(ValueError):
        P.BoundarySet(np.array([0, 1]), np.array([[0, 0, np.nan], [0, 0, 0]]), np.zeros((2, 3)))
    b = P.BoundarySet(np.array([2, 5]), np.zeros((2, 3)), np.zeros((2, 3)))
    assert b.position_of(5) == 1
    with pytest.raises(E.UnknownIndexError):
        b.position_of(3)


def test_error_hierarchy_mirrors_reference():
    for name in ("DuplicateNodesError", "NotPositiveDefiniteError", "DimensionMismatchError",
                 "EmptySupportSetError", "InvalidGroupCountError", "UnknownIndexError",
                 "EmptyGroupError", "TooFewBoundaryNodesError", "SelectionStalledError",
                 "InvalidCountError"):
        cls = getattr(E, name)
        assert issubclass(cls, E.RBFDeformError) and issubclass(cls, ValueError)


def test_host_helpers_match_reference_formulas():
    assert P.wendland_c2(0.5) == pytest.approx(0.1875, abs=1e-15)
    assert P.wendland_c2(np.array([0.0, 0.5, 1.0, 3.0])).tolist() == [1.0, 0.1875, 0.0, 0.0]
    with pytest.raises(ValueError):
        P.wendland_c2(-0.1)
    phi = P.assemble_phi([[0, 0, 0], [2.0, 0, 0]], 2.0)
    assert np.array_equal(phi, np.eye(2))
    with pytest.raises(E.DuplicateNodesError):
        P.assemble_phi([[0, 0, 0], [1, 1, 1], [0, 0, 0]], 2.0)


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    s = P.SupportSet(np.array([0]), np.zeros((1, 3)), np.ones((1, 3)))
    with pytest.raises(E.NativeUnavailableError):
        P.evaluate_displacements(np.zeros((4, 3)), s, 1.0)
    b = P.BoundarySet(np.arange(5), np.random.default_rng(0).normal(size=(5, 3)), np.ones((5, 3)))
    with pytest.raises(E.NativeUnavailableError):
        P.gcb_select(b, P.SelectionConfig(radius=1.0, tol=1e-6, max_supports=5))
    with pytest.raises(E.NativeUnavailableError):
        P.CholeskyState().append([1.0])


def test_native_pcg64_partition_is_numpy_bits():
    """rbf_partition (C++ host restatement of numpy's PCG64 permutation +
    round-robin deal) reproduces numpy bit for bit, incl. large nb where
    random_interval's rejection loop and the 32-bit buffering matter."""
    from paper_2004_04817_b200.selection import _partition_native

    rng = np.random.default_rng(2024)
    cases = [(3, 1, 0), (10, 3, 0), (20000, 32, 0), (80000, 48, 0), (200000, 64, 0)]
    cases += [(int(rng.integers(3, 5000)), 0, int(rng.integers(0, 2**63))) for _ in range(20)]
    for nb, m, seed in cases:
        m = m or int(rng.integers(1, nb + 1))
        flat, off = _partition_native(nb, m, seed)
        groups = O.partition(nb, m, seed)
        assert off[-1] == nb
        for j in range(m):
            assert np.array_equal(flat[off[j]:off[j + 1]], groups[j]), (nb, m, seed)
