"""The multi-GPU path (paper_2004_04817_b200.multi) end to end on the device
kernels, with two ranks (gloo) sharing the one GPU of the test box: the
loop on rank 0 with RBF_GCB_NO_SWEEP, the support broadcast, the sharded
final sweep (rbf_errors_argmax_dev per slice, all-gather of the 16-byte
records, rbf_best_fold on the device), the sharded error_summary and the
volume shards. No kernel waits on another rank (the collectives are host
side under gloo), so sharing one GPU is safe; under NCCL on N GPUs the same
code moves the records device to device.

Compared against the one-GPU path and the reference goldens: identical
support sequences and final-sweep node, maxima within 1e-12 relative of the
one-GPU sweep, volume shards bitwise equal to one launch."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import load_golden

pytestmark = pytest.mark.gpu
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
    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import _native as N
    from paper_2004_04817_b200 import multi
    from paper_2004_04817_b200 import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.config(0, nv=100_000)
        b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
        cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=8, seed=0)
        with N.launch_log() as log:
            res = multi.gcb_select(b, cfg)
        fs = res.history.final_sweep
        summ = multi.error_summary(b, res.support, wl.radius)
        shard, span = multi.deform_points(wl.volume, res.support, wl.radius, sharded_input=False)
        out = {"rank": rank, "seq": np.asarray(res.support.nodes), "weights": res.support.weights,
               "final": (fs.iteration, fs.node, fs.kernel_evals, fs.cum_kernel_evals),
               "final_max": fs.local_max_error, "converged": res.converged,
               "nrec": len(res.history.records), "summary": (summ.max_error, summ.rms_error, summ.node_of_max),
               "span": span, "shard": shard, "launches": dict(log.by_name)}
        q.put(out)
    except BaseException as exc:
        q.put({"rank": rank, "error": repr(exc)})
        raise
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def multi_results():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = sorted((q.get(timeout=600) for _ in range(world)), key=lambda r: r["rank"])
    for p in procs:
        p.join(timeout=120)
    for r in results:
        assert "error" not in r, r.get("error")
    for p in procs:
        assert p.exitcode == 0
    return results


def test_sharded_selection_matches_reference_golden(cuda, multi_results):
    g = load_golden("cfg0_m8")
    for r in multi_results:
        assert np.array_equal(r["seq"], g["seq"])
        assert r["final"][1] == int(g["final"][1])  # node of the final maximum
        assert r["final_max"] == pytest.approx(float(g["final_max"]), rel=1e-9)
        assert r["converged"] == bool(g["converged"])
    r0 = multi_results[0]
    assert list(r0["final"]) == g["final"].tolist()
    assert r0["nrec"] == len(g["rec_node"])
    assert multi_results[1]["nrec"] == 0  # non-src ranks: support set + final record only
    assert np.array_equal(multi_results[1]["weights"], r0["weights"])
    # the loop ran on rank 0 only; both ranks ran the sweep kernels and the fold
    assert r0["launches"].get("rbf_gcb_run", 0) >= 1
    assert multi_results[1]["launches"].get("rbf_gcb_run", 0) == 0
    assert all(r["launches"].get("rbf_best_fold") == 1 for r in multi_results)


def test_sharded_sweep_matches_one_gpu(cuda, multi_results):
    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import workloads as W

    wl = W.config(0, nv=100_000)
    b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
    cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=8, seed=0)
    one = P.gcb_select(b, cfg)
    r0 = multi_results[0]
    assert np.array_equal(np.asarray(one.support.nodes), r0["seq"])
    assert np.array_equal(one.support.weights, r0["weights"])  # same loop, same bits
    fs = one.history.final_sweep
    assert r0["final"][1] == fs.node
    assert r0["final_max"] == pytest.approx(fs.local_max_error, rel=1e-12)
    summ = P.error_summary(b, one.support, wl.radius)
    for r in multi_results:
        mx, rms, node = r["summary"]
        assert node == summ.node_of_max
        assert mx == pytest.approx(summ.max_error, rel=1e-12)
        assert rms == pytest.approx(summ.rms_error, rel=1e-12)


def test_volume_shards_bitwise(cuda, multi_results):
    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import workloads as W

    wl = W.config(0, nv=100_000)
    r0 = multi_results[0]
    s = P.SupportSet(r0["seq"], wl.points[r0["seq"]], r0["weights"])
    full = P.deform_points(wl.volume, s, wl.radius)
    joined = np.concatenate([r["shard"] for r in multi_results])
    assert [r["span"] for r in multi_results] == [(0, 50_000), (50_000, 100_000)]
    assert np.array_equal(joined, full)


def test_sweep_single_rank_and_empty_shards(cuda):
    """world = 1 (a plain process group of one) and a boundary smaller than
    the world: the empty shard contributes the neutral record."""
    import torch
    import torch.distributed as dist

    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import _native as N
    from paper_2004_04817_b200 import multi

    lib = N.require_cuda()
    rec = torch.empty(2, dtype=torch.float64, device="cuda")
    sp = torch.zeros((1, 3), dtype=torch.float64, device="cuda")
    N.check(lib.rbf_errors_argmax_dev(N.dptr(sp), N.dptr(sp), None, 0, N.dptr(sp), N.dptr(sp), 1, 1.0,
                                      None, 0, N.dptr(rec), N.dptr(sp), 8, N.stream_ptr()), "empty")
    assert rec.tolist() == [-1.0, 2147483647.0]
    recs = torch.tensor([[0.5, 7.0], [-1.0, 2147483647.0], [0.5, 3.0], [0.25, 1.0]],
                        dtype=torch.float64, device="cuda")
    out = torch.empty(2, dtype=torch.float64, device="cuda")
    N.check(lib.rbf_best_fold(N.dptr(recs), 4, N.dptr(out), N.stream_ptr()), "fold")
    assert out.tolist() == [0.5, 3.0]  # ties to the lowest position
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(3)
        pts = rng.normal(size=(300, 3))
        disp = rng.normal(size=(300, 3)) * 0.01
        b = P.BoundarySet(np.arange(300) * 2 + 5, pts, disp)
        s = P.SupportSet(b.indices[:20], pts[:20], rng.normal(size=(20, 3)) * 0.01)
        a = multi.error_summary(b, s, 1.5)
        e = P.error_summary(b, s, 1.5)
        assert (a.node_of_max, a.max_error, a.rms_error) == (e.node_of_max, e.max_error, e.rms_error)
    finally:
        dist.destroy_process_group()
