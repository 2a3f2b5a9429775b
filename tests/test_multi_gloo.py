"""world_size-2 gloo tests of the multi-GPU plumbing (paper_2004_04817_b200.multi)
on CPU: the support broadcast (count, then one packed buffer with the node
positions), the record all-gather, and the contiguous shards. The device
half of the same path (the sharded sweep's kernels and the device fold) is
driven end to end by tests/test_gpu_multi.py (two ranks sharing one GPU)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2004_04817_b200.multi import shard_range

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    sys.path.insert(0, REPO)
    from paper_2004_04817_b200 import multi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(5)
        sp = rng.normal(size=(57, 3))
        sw = rng.normal(size=(57, 3))
        nodes = rng.permutation(1000)[:57]
        if rank == 0:
            p, w, nd = multi.broadcast_support(torch.from_numpy(sp), sw, nodes=nodes)
        else:
            p, w, nd = multi.broadcast_support(None, None)
        ok_b = (np.array_equal(p.numpy(), sp) and np.array_equal(w.numpy(), sw)
                and np.array_equal(nd.numpy(), nodes))
        # a support set without node ids, and an empty one
        if rank == 0:
            _, _, none = multi.broadcast_support(sp[:3], sw[:3])
            pe, we, _ = multi.broadcast_support(np.zeros((0, 3)), np.zeros((0, 3)))
        else:
            _, _, none = multi.broadcast_support(None, None)
            pe, we, _ = multi.broadcast_support(None, None)
        ok_b = ok_b and none is None and pe.shape == (0, 3) and we.shape == (0, 3)
        rec = torch.tensor([float(rank) * 0.5 + 1.0, float(100 + rank)], dtype=torch.float64)
        rows = multi.all_gather_rows(rec)
        part, span = multi.shard_of(np.arange(1001))
        q.put((rank, ok_b, rows.numpy(), span, part[:2].tolist()))
    except BaseException as exc:  # report instead of leaving the parent waiting
        q.put((rank, repr(exc), None, None, None))
        raise
    finally:
        dist.destroy_process_group()


def test_gloo_multi_plumbing():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted((q.get(timeout=180) for _ in range(world)), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_b, rows, span, head in results:
        assert ok_b is True, ok_b
        assert rows.tolist() == [[1.0, 100.0], [1.5, 101.0]]
        assert span == shard_range(1001, rank, world)
        assert head == [span[0], span[0] + 1]


def test_shard_range_covers():
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans[:-1], spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1
            # rank 0 holds the largest shard (the sweep pads every shard to it)
            assert sizes[0] == max(sizes)


def test_bench_rejects_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=1" in r.stderr
