"""Multi-GPU sharding of the two stages that partition naturally
(SURVEY.md §8(e)): the volume evaluation (t3) and the all-boundary error
sweep (the selection's final sweep, reference selection.py:388-412, and
``error_summary``, reference metrics.py:77-88). The greedy loop itself is
sequential and stays on one GPU (``src``).

One process per GPU; ``torch.distributed`` (NCCL over NVLink / NVSwitch) is
the plumbing, the compute is this package's sm_100a kernels:

* ``broadcast_support``: the support set + weights (48 B per support, one
  packed (Nc, 7) float64 device buffer: point, weight, boundary position)
  from the rank that ran the loop to every rank;
* ``sweep``: every rank scans its contiguous slice of boundary rows with
  ``rbf_errors_argmax_dev`` (the fused error + arg-max kernel; its 16-byte
  (max error, position) record stays on the device), the records are
  all-gathered (``all_gather_into_tensor``, device to device) and folded on
  the device by ``rbf_best_fold`` (ties to the lowest position, reference
  selection.py:231-234) -- identical on every rank;
* ``gcb_select``: the reference's entry point with the loop on ``src``
  (``RBF_GCB_NO_SWEEP``: the loop kernel stops before its final sweep) and
  the final sweep sharded over all ranks;
* ``deform_points`` / ``deform_shard``: each rank deforms its contiguous
  shard of the volume. The kernel's per-target summation order does not
  depend on the launch, so the union of the shards is bitwise identical to
  a one-GPU run (no data-path collective).

The per-row error values of a sharded sweep agree with a one-GPU sweep to
rounding (the error kernel splits small scans over support slices, and a
shard is smaller than the whole boundary); the arg-max record is folded
exactly. With the gloo backend (CPU tests, tests/test_multi_gloo.py, or a
world-2 run sharing one GPU in tests/test_gpu_multi.py) CUDA tensors are
staged through host memory for the collective only.
"""

from dataclasses import replace

import numpy as np

from . import _native as N


def shard_range(n, rank, world):
    """Contiguous [lo, hi) slice of n items owned by ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _dist():
    import torch.distributed as dist

    return dist


def _rank_world(group):
    dist = _dist()
    return dist.get_rank(group), dist.get_world_size(group)


def _staged(tensor, group):
    """gloo cannot run every collective on CUDA tensors: stage through host."""
    return tensor.is_cuda and _dist().get_backend(group) == "gloo"


def broadcast_(tensor, src=0, group=None):
    """In-place broadcast of a tensor (device to device under NCCL)."""
    dist = _dist()
    if _staged(tensor, group):
        h = tensor.cpu()
        dist.broadcast(h, src=src, group=group)
        tensor.copy_(h)
    else:
        dist.broadcast(tensor, src=src, group=group)
    return tensor


def all_gather_rows(rec, group=None):
    """(world, *rec.shape) tensor of every rank's ``rec`` (equal shapes)."""
    t = N.torch()
    dist = _dist()
    world = dist.get_world_size(group)
    src = rec.contiguous().reshape(-1)
    if _staged(rec, group):
        src = src.cpu()
    out = t.empty(world * src.numel(), dtype=rec.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.reshape(world, *rec.shape).to(rec.device)


def broadcast_support(points, weights, src=0, group=None, nodes=None):
    """Broadcast (Nc, 3) points and weights (and, optionally, the (Nc,)
    support node ids) from ``src``: the count first, then one packed
    (Nc, 7) float64 buffer. ``points`` / ``weights`` are tensors on every
    rank's device on ``src`` (numpy accepted) and ignored elsewhere.
    Returns (points, weights, nodes) device tensors on every rank; nodes is
    an int64 tensor (or None when ``src`` passed none)."""
    t = N.torch()
    dist = _dist()
    dev = t.device("cuda", t.cuda.current_device()) if t.cuda.is_available() else t.device("cpu")
    rank = dist.get_rank(group)
    head = t.zeros(2, dtype=t.int64, device=dev)
    if rank == src:
        head[0] = int(points.shape[0])
        head[1] = 1 if nodes is not None else 0
    broadcast_(head, src=src, group=group)
    nc, has_nodes = (int(v) for v in head.tolist())
    buf = t.empty((nc, 7), dtype=t.float64, device=dev)
    if rank == src and nc:
        buf[:, 0:3] = t.as_tensor(points, dtype=t.float64).to(dev)
        buf[:, 3:6] = t.as_tensor(weights, dtype=t.float64).to(dev)
        buf[:, 6] = (t.as_tensor(np.asarray(nodes, dtype=np.float64)).to(dev) if has_nodes
                     else 0.0)
    broadcast_(buf, src=src, group=group)
    nodes_out = buf[:, 6].to(t.int64) if has_nodes else None
    return buf[:, 0:3].contiguous(), buf[:, 3:6].contiguous(), nodes_out


class SweepResult:
    """(max error, position of the max, errors or None) of a sharded sweep."""

    __slots__ = ("max_error", "pos", "errors")

    def __init__(self, max_error, pos, errors):
        self.max_error, self.pos, self.errors = max_error, pos, errors


def sweep(points, disp, support_points, weights, radius, group=None, want_errors=False):
    """Sharded all-boundary error sweep on device tensors.

    ``points`` / ``disp``: the whole boundary (Nb, 3) on every rank's device
    (each rank reads only its slice); ``support_points`` / ``weights``
    (Nc, 3) device tensors (``broadcast_support``). Each rank scans rows
    [lo, hi) with the fused error + arg-max kernel, the 16-byte records
    are all-gathered and folded on the device. ``want_errors`` also
    all-gathers the per-row errors (padded to the largest shard) and
    returns the full (Nb,) vector on every rank."""
    lib = N.require_cuda()
    t = N.torch()
    rank, world = _rank_world(group)
    nb = points.shape[0]
    lo, hi = shard_range(nb, rank, world)
    n = hi - lo
    dev = points.device
    rec = t.empty(2, dtype=t.float64, device=dev)
    span = shard_range(nb, 0, world)[1]  # largest shard (rank 0's)
    err = t.empty(span, dtype=t.float64, device=dev) if want_errors else None
    if want_errors and n < span:
        err[n:] = 0.0
    nbytes = lib.rbf_errors_scratch_bytes(max(n, 1))
    scratch = t.empty(nbytes, dtype=t.uint8, device=dev)
    pts = points[lo:hi]
    dsp = disp[lo:hi]
    with N.launching("rbf_errors_argmax", kernels=3 if n else 1):
        rc = lib.rbf_errors_argmax_dev(
            N.dptr(pts) if n else N.dptr(points), N.dptr(dsp) if n else N.dptr(disp), None, n,
            N.dptr(support_points), N.dptr(weights), support_points.shape[0], float(radius),
            N.dptr(err) if err is not None else None, lo, N.dptr(rec), N.dptr(scratch), nbytes,
            N.stream_ptr())
    N.check(rc, "rbf_errors_argmax_dev")
    recs = all_gather_rows(rec, group)
    best = t.empty(2, dtype=t.float64, device=dev)
    with N.launching("rbf_best_fold", kernels=1):
        rc = lib.rbf_best_fold(N.dptr(recs), world, N.dptr(best), N.stream_ptr())
    N.check(rc, "rbf_best_fold")
    errors = None
    if want_errors:
        rows = all_gather_rows(err, group).cpu().numpy()
        errors = np.concatenate([rows[r, : hi_ - lo_] for r, (lo_, hi_) in
                                 enumerate(shard_range(nb, q, world) for q in range(world))])
    e, p = best.tolist()
    return SweepResult(float(e), int(p), errors)


def gcb_select(boundary, config, group=None, src=0):
    """Collective ``gcb_select`` (reference selection.py:257-271): every rank
    of ``group`` calls it with the same boundary and config. The loop runs
    on ``src`` (one GPU, the reference's sequential dependency), the final
    sweep is sharded over all ranks. Returns the SelectionResult on every
    rank: on ``src`` with the full history, elsewhere with the support set,
    the final sweep record and ``converged`` (``history.records`` empty)."""
    import time

    from .core import SupportSet
    from .selection import IterationRecord, SelectionHistory, SelectionResult, _boundary_on_device, _gcb_run

    t = N.torch()
    rank, world = _rank_world(group)
    res = _gcb_run(boundary, config, sweep=False) if rank == src else None
    if rank == src:
        sp, sw, nodes = broadcast_support(res.support.points, res.support.weights, src, group,
                                          nodes=np.searchsorted(boundary.indices, res.support.nodes))
    else:
        sp, sw, nodes = broadcast_support(None, None, src, group)
    pts, disp = _boundary_on_device(boundary)
    t.cuda.synchronize()
    t0 = time.perf_counter()
    swr = sweep(pts, disp, sp, sw, config.radius, group)
    t1 = time.perf_counter() - t0
    node = int(boundary.indices[swr.pos])
    converged = swr.max_error <= config.tol
    if rank == src:
        res.history.final_sweep = replace(res.history.final_sweep, node=node,
                                          local_max_error=swr.max_error, t1_s=t1)
        return replace(res, converged=converged)
    pos = nodes.cpu().numpy()
    n = len(pos)
    hist = SelectionHistory(seed=config.seed, m=config.m)
    hist.final_sweep = IterationRecord(iteration=-1, group=-1, node=node, local_max_error=swr.max_error,
                                       kernel_evals=len(boundary) * n, cum_kernel_evals=-1, t1_s=t1,
                                       t2_s=0.0)
    support = SupportSet(nodes=boundary.indices[pos], points=boundary.points[pos], weights=sw.cpu().numpy())
    return SelectionResult(support=support, history=hist, converged=converged)


def error_summary(boundary, support, radius, group=None):
    """Collective ``error_summary`` (reference metrics.py:77-88): the
    boundary sweep sharded over the ranks; every rank returns the same
    ErrorSummary. The RMS is the reference's numpy expression over the
    gathered per-row errors."""
    from .core import _to_device
    from .errors import EmptySupportSetError
    from .metrics import ErrorSummary
    from .selection import _boundary_on_device

    if len(support) == 0:
        raise EmptySupportSetError("support set is empty")
    pts, disp = _boundary_on_device(boundary)
    sp = _to_device(support.points)
    w = _to_device(support.weights)
    res = sweep(pts, disp, sp, w, radius, group, want_errors=True)
    errors = res.errors
    rms = float(np.sqrt(np.mean(errors * errors)))
    return ErrorSummary(max_error=res.max_error, rms_error=rms, node_of_max=int(boundary.indices[res.pos]))


def shard_of(points, group=None):
    """This rank's contiguous shard of ``points`` (numpy or tensor) and its
    [lo, hi) range."""
    rank, world = _rank_world(group)
    lo, hi = shard_range(len(points), rank, world)
    return points[lo:hi], (lo, hi)


def deform_shard(points, support_points, weights, radius, out=None):
    """Device-resident deformation of this rank's shard (torch tensors;
    ``support_points`` / ``weights`` from ``broadcast_support``)."""
    from .core import eval_device

    return eval_device(points, support_points, weights, radius, deform=True, out=out)


def deform_points(points, support, radius, group=None, sharded_input=True):
    """Collective ``deform_points`` (reference core.py:359-367): with
    ``sharded_input`` each rank passes its own shard and gets it back
    deformed (no collective at all: the support set must already be on every
    rank); otherwise every rank passes the whole volume and gets its own
    shard's result and range."""
    from .core import deform_points as deform

    if sharded_input:
        return deform(points, support, radius)
    shard, span = shard_of(points, group)
    return deform(shard, support, radius), span
