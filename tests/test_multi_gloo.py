"""world_size-2 gloo tests of the multi-GPU plumbing (paper_2004_04817_b200.multi)
on CPU: support broadcast, contiguous target shards whose union equals the
single-process result bit for bit, and the (max, lowest position) combine.
The compute callable is the CPU oracle here (tests only)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2004_04817_b200.multi import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.join(here, "..", "oracle"))
    sys.path.insert(0, os.path.join(here, ".."))
    import rbf_oracle as O
    from paper_2004_04817_b200 import multi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        sp = rng.normal(size=(57, 3))
        sw = rng.normal(size=(57, 3))
        vol = rng.normal(size=(1001, 3)) * 1.5
        if rank == 0:
            p, w = multi.broadcast_support(torch.from_numpy(sp), torch.from_numpy(sw))
        else:
            p, w = multi.broadcast_support(None, torch.zeros((0, 3), dtype=torch.float64))
        assert np.array_equal(p.numpy(), sp) and np.array_equal(w.numpy(), sw)

        def evaluate(v, s, ww, r, deform):
            u = O.eval_sum(v.numpy(), s.numpy(), ww.numpy(), r)
            return torch.from_numpy(v.numpy() + u if deform else u)

        lo, hi, shard = multi.deform_sharded(torch.from_numpy(vol), p, w, 2.0, evaluate, rank, world)
        parts = [None] * world
        dist.all_gather_object(parts, (lo, hi, shard.numpy()))
        # a sweep: per-rank (max, lowest pos) over a shared error vector with ties
        errs = np.array([0.5, 2.0, 1.0, 2.0, 0.1, 2.0, 0.3])

        def errors_of(a, b):
            if a == b:
                return -1.0, 1 << 30
            seg = errs[a:b]
            k = int(np.flatnonzero(seg == seg.max())[0])
            return float(seg[k]), a + k

        best = multi.sweep_sharded(len(errs), errors_of, rank, world)
        q.put((rank, parts, best))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_sharded_volume_and_sweep(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "oracle"))
    import rbf_oracle as O

    rng = np.random.default_rng(5)
    sp = rng.normal(size=(57, 3))
    sw = rng.normal(size=(57, 3))
    vol = rng.normal(size=(1001, 3)) * 1.5
    full = vol + O.eval_sum(vol, sp, sw, 2.0)
    for rank, parts, best in results:
        joined = np.concatenate([s for _, _, s in sorted(parts, key=lambda t: t[0])])
        # the CPU oracle's BLAS blocking depends on the span layout, so shards
        # agree to rounding here; the GPU kernel is bitwise shard-invariant
        # (tests/test_gpu_parity.py::test_eval_shards_are_bitwise_identical)
        assert np.abs(joined - full).max() <= 1e-13 * np.abs(full).max()
        assert [(lo, hi) for lo, hi, _ in parts] == [shard_range(1001, r, world) for r in range(world)]
        assert best == (2.0, 1)


def test_shard_range_covers():
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans[:-1], spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
