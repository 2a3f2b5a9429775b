"""Boundary metrics on the GPU: nearest-support distances, the KL divergence
between support distributions, and interpolation-error summaries and
histories (reference ``metrics.py:14-115``).

The mesh-cell quality metrics of the reference module (``cell_quality``,
``quality_report``) are surface-mesh analytics outside the hot path and are
not part of this package.
"""

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .core import CholeskyState, SupportSet, _device, _to_device, _to_host
from .errors import EmptySupportSetError
from .selection import _argmax_lowest_id, _errors_at

# Floor for the reference distance in the KL ratio (metrics.py:14-16).
KL_DISTANCE_FLOOR = 1e-12


@dataclass(eq=False)
class ErrorSummary:
    """Maximum and RMS interpolation error over the boundary (metrics.py:21-27)."""

    max_error: float
    rms_error: float
    node_of_max: int


def _nearest_device(points, support_points):
    """min_i |p_k - s_i| for every row of ``points`` (device kernel
    ``rbf_nearest``: cdist's rounding, so bit-identical to the reference)."""
    lib = N.require_cuda()
    t = N.torch()
    pts = _to_device(np.ascontiguousarray(points, dtype=float).reshape(-1, 3))
    sp = _to_device(np.ascontiguousarray(support_points, dtype=float).reshape(-1, 3))
    out = t.empty(pts.shape[0], dtype=t.float64, device=_device())
    with N.launching("rbf_nearest", kernels=1 if pts.shape[0] else 0):
        rc = lib.rbf_nearest(N.dptr(pts), pts.shape[0], N.dptr(sp), sp.shape[0], N.dptr(out),
                             N.stream_ptr())
    N.check(rc, "rbf_nearest")
    return _to_host(out)


def _nearest_distances(support, boundary):
    """Distance from every boundary node to its closest support (metrics.py:45-48)."""
    if len(support) == 0:
        raise EmptySupportSetError("support set is empty")
    return _nearest_device(boundary.points, support.points)


def nearest_support_distance(index, support, boundary):
    """Distance from boundary node ``index`` to the closest support node
    (metrics.py:51-60); the same kernel as the all-nodes scan, so the two
    agree bit for bit."""
    if len(support) == 0:
        raise EmptySupportSetError("support set is empty")
    pos = boundary.position_of(index)
    return float(_nearest_device(boundary.points[pos][None, :], support.points)[0])


def kl_divergence(s1, s2, boundary):
    """sum d1 log(d1 / max(d2, 1e-12)) over boundary nodes with d1 > 0
    (metrics.py:63-74). Distances from the device, bit-identical to the
    reference's; the final sum is the reference's numpy expression."""
    d1 = _nearest_distances(s1, boundary)
    d2 = np.maximum(_nearest_distances(s2, boundary), KL_DISTANCE_FLOOR)
    mask = d1 > 0.0
    return float(np.sum(d1[mask] * np.log(d1[mask] / d2[mask])))


def error_summary(boundary, support, radius):
    """Scan every boundary node (one fused device pass) and summarise the
    residuals (metrics.py:77-88)."""
    errors = _errors_at(np.arange(len(boundary)), boundary, support.points, support.weights, radius)
    worst = _argmax_lowest_id(errors, boundary.indices)
    rms = float(np.sqrt(np.mean(errors * errors)))
    return ErrorSummary(max_error=float(errors[worst]), rms_error=rms,
                        node_of_max=int(boundary.indices[worst]))


def error_history(boundary, support_nodes, radius, every=50):
    """Error summaries at prefixes of a support sequence (metrics.py:91-115).

    The reference re-factors every sampled prefix one-shot (``cho_factor``);
    here the sequence is factored once by device appends (rows built on the
    device, one host round trip for the whole sequence) and every prefix is
    solved with the leading block of that factor (a prefix of the packed
    triangles), then the boundary is scanned on the device. Same
    mathematics; agreement is at the factorisation's rounding level.
    """
    support_nodes = np.asarray(support_nodes, dtype=np.intp)
    total = len(support_nodes)
    counts = list(range(every, total, every))
    if not counts or counts[-1] != total:
        counts.append(total)
    positions = np.searchsorted(boundary.indices, support_nodes)
    pts_all = boundary.points[positions]
    state = CholeskyState()
    state._append_points(pts_all, radius)  # every row on the device, one host round trip
    out = []
    for n in counts:
        if n == 0:
            weights = np.zeros((0, 3))
        else:
            weights = state._solve_prefix(boundary.disp[positions[:n]], n)
        prefix = SupportSet(nodes=support_nodes[:n], points=pts_all[:n], weights=weights)
        out.append((n, error_summary(boundary, prefix, radius)))
    return out
