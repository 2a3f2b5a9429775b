"""Multi-GPU sharding of the two stages that partition naturally
(SURVEY.md §8(e)): the volume evaluation (t3) and the all-boundary error
sweep. One process per GPU; torch.distributed (NCCL over NVLink/NVSwitch)
is the plumbing:

* the support set + weights (48 B per support) are broadcast from the rank
  that ran the selection loop (the loop itself stays on one GPU);
* targets are split into contiguous shards, one per rank, with no
  data-path collective -- each rank evaluates its shard with the same
  kernel, whose per-target summation order does not depend on the shard,
  so the union of the shards is bitwise identical to a one-GPU run;
* a sharded sweep combines per-rank (max error, lowest position) records
  with one all-gather of 16 B per rank.

The compute callables are parameters so the collective logic can be
exercised on CPU with the gloo backend (tests/test_multi_gloo.py).
"""

import numpy as np


def shard_range(n, rank, world):
    """Contiguous [lo, hi) slice of n items owned by ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def broadcast_support(points, weights, src=0, group=None):
    """Broadcast (Nc, 3) points and weights from ``src`` (one packed
    (Nc, 6) float64 buffer plus its length). Tensors on the backend's
    device; returns (points, weights) on every rank."""
    import torch
    import torch.distributed as dist

    dev = points.device if points is not None else weights.device
    n = torch.tensor([0 if points is None else points.shape[0]], dtype=torch.int64, device=dev)
    dist.broadcast(n, src=src, group=group)
    buf = torch.empty((int(n.item()), 6), dtype=torch.float64, device=dev)
    if dist.get_rank() == src:
        buf[:, :3] = points
        buf[:, 3:] = weights
    dist.broadcast(buf, src=src, group=group)
    return buf[:, :3].contiguous(), buf[:, 3:].contiguous()


def combine_best(err, pos, group=None):
    """Global (max err, lowest position) over ranks: all-gather of one
    16-byte record per rank, folded identically everywhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = err.device
    rec = torch.stack([err.to(torch.float64), pos.to(torch.float64)]).reshape(1, 2)
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec, group=group)
    allrec = torch.cat(out).cpu().numpy()
    best_e, best_p = -1.0, np.inf
    for e, p in allrec:
        if e > best_e or (e == best_e and p < best_p):
            best_e, best_p = e, p
    return float(best_e), int(best_p)


def deform_sharded(volume, support_points, weights, radius, evaluate, rank, world, deform=True):
    """Evaluate this rank's contiguous shard of ``volume`` with ``evaluate``
    (the device kernel on GPUs). Returns (lo, hi, result_shard)."""
    lo, hi = shard_range(volume.shape[0], rank, world)
    return lo, hi, evaluate(volume[lo:hi], support_points, weights, radius, deform)


def sweep_sharded(nb, errors_of, rank, world, group=None):
    """Sharded all-boundary error sweep: ``errors_of(lo, hi)`` returns this
    rank's (max err, position) over boundary rows [lo, hi)."""
    import torch

    lo, hi = shard_range(nb, rank, world)
    e, p = errors_of(lo, hi)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else "cpu"
    return combine_best(torch.tensor(e, device=dev), torch.tensor(p, device=dev), group=group)
