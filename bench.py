#!/usr/bin/env python
"""Benchmark: one GCB-greedy selection + volume deformation per step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

A step is the reference's hot path on one batch of synthetic input
(BASELINE.json configs[C], default C = 1: Nb = 20,000 wing nodes,
Nv = 2,000,000 volume nodes, GCB m = 32, R = 2, tol = 1e-4 max|d|, FP64):
the full selection loop including the final sweep (device resident)
followed by deform_points over all Nv volume nodes.

N > 1 GPUs: one process per GPU. Without WORLD_SIZE in the environment,
``--gpus N`` re-launches itself under ``torch.distributed.run`` with N
ranks (127.0.0.1); under torchrun WORLD_SIZE must equal N. The default
multi-GPU step is the sharded one north_star describes (``--multi shard``,
strong scaling: the whole job is one selection + one Nv volume): the loop
runs on rank 0, the support set is broadcast (NCCL), the final sweep and the
volume are split into contiguous shards; ``volume_ms`` is
the volume stage's max over ranks and ``volume_speedup`` divides the
one-GPU volume time (measured in the same run on rank 0) by it.
``--multi replicas`` runs N independent whole steps instead (weak scaling).

Metric: RBF pair-evaluations per second, whole job, with
pairs = sum_i card(G_i) * Nc(i) + Nb * Nc   (selection, = cum_kernel_evals)
      + Nv * Nc                              (volume).
`value` times device-resident inputs with CUDA events; `e2e` times the same
step through the public API with host (pinned) buffers, host<->device copies
inside the timed region. L2 (126 MB) is flushed between timed steps by
writing a 256 MiB buffer. Rank 0 prints ONE JSON line on stdout.

--impl reference times the reference algorithm on the host CPU (the oracle
port in oracle/, all host cores): per step the full selection loop plus a
strided sample of the volume, the volume time scaled to all Nv targets, so
its pairs/s is quoted on the same pair mix as the GPU arm.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

FLOP_PER_PAIR = 22  # 3 sub, 5 r^2, 1 sqrt, 1 div, 1 sub, 2 mul, 2 (4eta+1), 1 mul, 6 acc
METRIC = "RBF pair-evals/s (GCB error + volume deform)"
UNIT = "pair-evals/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=100_000, help="volume targets in the CPU sample")
    ap.add_argument("--multi", choices=["shard", "replicas"], default="shard",
                    help="N > 1: selection on rank 0 + final sweep and volume sharded over the ranks "
                         "(default, strong scaling) or N independent whole steps (weak scaling)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(cfg):
    from paper_2004_04817_b200 import workloads as W

    return W.config(cfg)


def multi_mode(args, world):
    return "single" if world == 1 else args.multi


def relaunch(args):
    """``--gpus N`` outside torchrun: run this script under
    torch.distributed.run with N ranks, one per GPU (127.0.0.1)."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(REPO / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def tol_frac(wl):
    return wl.tol / float(np.linalg.norm(wl.disp, axis=1).max())


def config_desc(wl, world, extra=None, mode="single"):
    d = {
        "workload": f"BASELINE configs[{wl.name[-1]}]: {wl.name}, Nb={wl.nb}, Nv={wl.nv}, "
                    f"GCB m={wl.m}, R={wl.radius}, tol={tol_frac(wl):.0e}*max|d|, seed={wl.seed}",
        "nb": wl.nb,
        "nv": wl.nv,
        "m": wl.m,
        "radius": wl.radius,
        "tol": wl.tol,
        "parallelism": ("1 GPU" if mode == "single" else
                        f"{world} independent replicas (each GPU runs the whole step)"
                        if mode == "replicas" else
                        f"selection loop on rank 0; final sweep and volume sharded over {world} GPUs"),
        "l2": "flushed between timed steps (256 MiB write)",
    }
    if extra:
        d.update(extra)
    return d


# ----------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def _target(self):
        import torch

        try:
            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return uuid if uuid.startswith("GPU-") else "GPU-" + uuid
        except Exception:
            return str(self.device)

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20", "-i", self._target()],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        self.lines += [ln for ln in out.splitlines() if ln.strip()]
        self.proc = None

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = sorted(sm)[len(sm) // 2:]  # upper half = under load
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ peaks
def measure_fp64_peak():
    """FP64 peak on this GPU: best of our DFMA probe and cuBLAS DGEMM."""
    import ctypes

    import torch

    from paper_2004_04817_b200 import _native as N

    lib = N.require_cuda()
    dev = torch.cuda.current_device()
    scratch = torch.empty(lib.rbf_fp64_probe_scratch_bytes(dev), dtype=torch.uint8, device="cuda")
    flops = ctypes.c_double(0)
    best_probe = 0.0
    for iters in (2000, 20000, 20000, 20000):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        N.check(lib.rbf_fp64_probe(iters, N.dptr(scratch), ctypes.byref(flops), N.stream_ptr()), "probe")
        e1.record()
        torch.cuda.synchronize()
        best_probe = max(best_probe, flops.value / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    best_gemm = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best_gemm = max(best_gemm, 2 * 8192**3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    return {"fp64_dfma_probe_tflops": round(best_probe, 3), "fp64_dgemm_tflops": round(best_gemm, 3),
            "peak_tflops": round(max(best_probe, best_gemm), 3),
            "nominal_tflops": 37.0,
            "source": "measured in this run: max(DFMA probe, cuBLAS DGEMM 8192^3); "
                      "MEASURED_PEAKS.json has no FP64 entry"}


def load_traffic():
    p = REPO / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except Exception:
            return {}
    return {}


# ---------------------------------------------------------- CPU baseline
def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_oracle_step(wl, threads, sample):
    """One CPU step of the reference algorithm (the oracle port, numpy/scipy/
    OpenBLAS with the reference's own thread pool of ``threads`` workers):
    the full selection loop, then a strided ``sample`` of the volume whose
    time is scaled to all Nv targets (per-target cost is uniform: every
    target walks all Nc supports, reference core.py:301-334). The step's
    pairs are the GPU arm's: A_sel + Nv * Nc."""
    sys.path.insert(0, str(REPO / "oracle"))
    import rbf_oracle as O

    t0 = time.perf_counter()
    out = O.select(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, wl.m, wl.seed, threads=threads)
    t1 = time.perf_counter()
    idx = np.linspace(0, wl.nv - 1, min(sample, wl.nv)).astype(np.int64)
    O.eval_sum(wl.volume[idx], wl.points[out["seq"]], out["weights"], wl.radius, threads=threads)
    t2 = time.perf_counter()
    nc = len(out["seq"])
    sel_pairs = sum(r[4] for r in out["records"]) + out["final"][3]
    vol_s = (t2 - t1) * wl.nv / len(idx)
    return {"pairs": sel_pairs + wl.nv * nc, "seconds": (t1 - t0) + vol_s, "select_s": t1 - t0,
            "volume_sample_s": t2 - t1, "volume_s": vol_s, "nc": nc, "sample": len(idx),
            "selection_pairs": sel_pairs, "wall_s": t2 - t0}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_sample_desc(wl, s, threads):
    return (f"full selection loop (Nb={wl.nb}, m={wl.m}, {s['select_s']:.2f} s) + {s['sample']} of {wl.nv} "
            f"volume targets ({s['volume_sample_s']:.2f} s, scaled x{wl.nv / s['sample']:.0f} to all Nv), "
            f"oracle port of the reference (numpy/scipy/OpenBLAS), {threads} thread(s), {cpu_model()}")


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    wl = workload(args.config)
    threads = host_threads()
    for _ in range(max(args.warmup, 0)):
        cpu_oracle_step(wl, threads, args.cpu_sample)
    steps = [cpu_oracle_step(wl, threads, args.cpu_sample) for _ in range(args.steps)]
    pairs = sum(s["pairs"] for s in steps)
    secs = sum(s["seconds"] for s in steps)
    value = pairs / secs
    one = cpu_oracle_step(wl, 1, args.cpu_sample)  # the workers = 1 leg
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / len(steps) * 1e3, "higher_is_better": True,
        "scaling": "weak" if multi_mode(args, world) == "replicas" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, "
                                                      "paper_2004_04817_b200/workloads.py)",
        "impl": "reference",
        "config": config_desc(wl, world, mode=multi_mode(args, world)),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": cpu_sample_desc(wl, steps[0], threads), "cpu_model": cpu_model()},
        "cpu_baseline_1_worker": {"value": one["pairs"] / one["seconds"], "unit": UNIT, "cores": 1,
                                  "kind": "port", "ms_per_step": one["seconds"] * 1e3,
                                  "sample": cpu_sample_desc(wl, one, 1)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "breakdown": {"select_s": statistics.mean(s["select_s"] for s in steps),
                      "volume_s": statistics.mean(s["volume_s"] for s in steps),
                      "volume_sample_s": statistics.mean(s["volume_sample_s"] for s in steps),
                      "nc": steps[0]["nc"], "selection_pairs": steps[0]["selection_pairs"],
                      "volume_pairs": wl.nv * steps[0]["nc"]},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------- GPU arm
def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import _native as N
    from paper_2004_04817_b200 import multi

    # RBF_BENCH_SHARE_GPU=1 (code-path check on a one-GPU box, with RBF_BENCH_BACKEND=gloo:
    # no kernel waits on another rank): every rank on device 0; numbers are not a measurement
    if os.environ.get("RBF_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group(os.environ.get("RBF_BENCH_BACKEND", "nccl"),
                                device_id=torch.device("cuda", local))
    N.require_cuda()

    def barrier():
        if world > 1:
            dist.barrier()

    wl = workload(args.config)
    peak = measure_fp64_peak()
    mode = multi_mode(args, world)
    replicas = mode == "replicas"
    shard = mode == "shard"
    boundary = P.stage_boundary(P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp))
    bpts, bdisp = boundary._device[2], boundary._device[3]
    cfg = P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=wl.m, seed=wl.seed)
    lo, hi = multi.shard_range(wl.nv, rank, world) if shard else (0, wl.nv)
    nv_local = hi - lo
    vol_d = torch.from_numpy(np.ascontiguousarray(wl.volume[lo:hi])).cuda()
    out_d = torch.empty_like(vol_d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    from paper_2004_04817_b200.selection import _gcb_run

    def device_step():
        """One step on device-resident inputs; returns (result or None, Nc)."""
        if not shard:  # the volume kernel queued behind the loop (select_and_deform)
            res, _ = P.select_and_deform(boundary, cfg, vol_d, out=out_d)
            return res, len(res.support)
        else:
            res = _gcb_run(boundary, cfg, sweep=False) if rank == 0 else None
            sp, sw, _ = (multi.broadcast_support(res.support.points, res.support.weights) if rank == 0
                         else multi.broadcast_support(None, None))
            sweep = multi.sweep(bpts, bdisp, sp, sw, wl.radius)
            if res is not None:
                res.history.final_sweep = replace(res.history.final_sweep, node=int(sweep.pos),
                                                  local_max_error=sweep.max_error)
        P.eval_device(vol_d, sp, sw, wl.radius, deform=True, out=out_d)
        return res, sp.shape[0]

    for _ in range(args.warmup):
        device_step()
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    times, logs, nc, a_sel, res = [], [], None, None, None
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with N.launch_log(timing=True) as log:
            e0.record()
            r, nc = device_step()
            e1.record()
        torch.cuda.synchronize()
        barrier()
        times.append(e0.elapsed_time(e1) * 1e-3)
        logs.append(log)
        if r is not None:
            res = r
            a_sel = r.history.final_sweep.cum_kernel_evals
    # e2e through the public API: host (pinned) buffers in and out
    vol_host_t = torch.from_numpy(np.ascontiguousarray(wl.volume[lo:hi])).pin_memory()
    vol_host = vol_host_t.numpy()
    from paper_2004_04817_b200 import selection as S

    def e2e_step(vol):
        """The public API from host arrays: a fresh BoundarySet (uploaded by the
        call), the partition recomputed (its cache cleared: the reference
        re-partitions on every call), the volume in and the result out."""
        with S._cache_lock:
            S._part_cache.clear()
        b_host = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
        if shard:
            sup = multi.gcb_select(b_host, cfg).support
            return sup, P.deform_points(vol, sup, wl.radius)
        res, moved = P.select_and_deform(b_host, cfg, vol)  # volume pipeline queued behind the loop
        return res.support, moved

    e2e_times = []
    for i in range(args.warmup + args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sup, moved = e2e_step(vol_host)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        barrier()
        if i >= args.warmup:
            e2e_times.append(t1 - t0)
    # the same with the volume as a plain (pageable) numpy array, as reference
    # API callers pass it: reported beside e2e, not instead of it
    vol_pageable = np.ascontiguousarray(wl.volume[lo:hi])
    e2e_pageable = []
    for i in range(args.warmup + min(args.steps, 5)):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_step(vol_pageable)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        barrier()
        if i >= args.warmup:
            e2e_pageable.append(t1 - t0)
    clocks.stop()
    assert moved.shape == (nv_local, 3)

    # per-phase device cycles of the selection loop: one extra, untimed run
    # with the phase clock on (it costs ~4 % of the loop, so the timed runs
    # leave it off)
    prof_hist = None
    if rank == 0:
        prof_hist = _gcb_run(boundary, cfg, phases=True).history

    # volume stage alone: this rank's shard (max over ranks) and, on rank 0,
    # the whole Nv on one GPU, for the volume-stage speed-up
    sp_d = torch.from_numpy(np.ascontiguousarray(sup.points)).cuda()
    sw_d = torch.from_numpy(np.ascontiguousarray(sup.weights)).cuda()

    def time_eval(v, o, reps=5):
        best = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            P.eval_device(v, sp_d, sw_d, wl.radius, deform=True, out=o)
            e1.record()
            torch.cuda.synchronize()
            best.append(e0.elapsed_time(e1))
        return statistics.median(best)

    barrier()
    vol_shard_ms = time_eval(vol_d, out_d)
    vol_full_ms = None
    if world > 1 and shard and rank == 0:
        del out_d
        full_d = torch.from_numpy(wl.volume).cuda()
        vol_full_ms = time_eval(full_d, torch.empty_like(full_d), reps=3)
        del full_d

    # ---- aggregate (max over ranks) ----
    t_local = float(sum(times))
    e2e_local = float(sum(e2e_times))
    e2e_pg_local = float(statistics.median(e2e_pageable))
    if world > 1:
        tt = torch.tensor([t_local, e2e_local, vol_shard_ms, e2e_pg_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total, e2e_total, vol_shard_max, e2e_pg = tt.tolist()
        a = torch.tensor([a_sel or 0], dtype=torch.int64, device="cuda")
        dist.broadcast(a, src=0)
        a_sel = int(a.item())
    else:
        t_total, e2e_total, vol_shard_max, e2e_pg = t_local, e2e_local, vol_shard_ms, e2e_pg_local
    pairs_per_step = (a_sel + wl.nv * nc) * (world if replicas else 1)
    value = pairs_per_step * args.steps / t_total
    e2e_value = pairs_per_step * args.steps / e2e_total

    # per-kernel device times (rank 0 view), roofline of the dominant kernel
    # per step: the selection may take several launches (capacity growth or
    # a switch of storage path), the volume one
    sel_ms = [sum(lg.kernel_ms("rbf_gcb_run")) for lg in logs if lg.kernel_ms("rbf_gcb_run")]
    vol_ms = [sum(lg.kernel_ms("rbf_eval")) for lg in logs if lg.kernel_ms("rbf_eval")]
    sweep_ms = [sum(lg.kernel_ms("rbf_errors_argmax")) for lg in logs if lg.kernel_ms("rbf_errors_argmax")]
    launches = sum(lg.count for lg in logs) / len(logs)
    launches_sel = sum(lg.by_name.get("rbf_gcb_run", 0) for lg in logs) / len(logs)
    traffic = {k: v.get("bytes_per_launch") for k, v in load_traffic().items()}
    peak_tf = peak["peak_tflops"]
    kernels = []
    if sel_ms:
        t = statistics.mean(sel_ms) * 1e-3
        sel_pairs = a_sel - (wl.nb * nc if shard and world > 1 else 0)
        ach = FLOP_PER_PAIR * sel_pairs / t / 1e12
        kernels.append({"kernel": "gcb_*_kernel (selection loop, launches per step: %d)"
                                  % round(launches_sel), "ms": t * 1e3,
                        "bound": "latency (dependent DSMEM hops / grid barriers)", "achieved": ach,
                        "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf,
                        "traffic": traffic.get("gcb_kernel")})
    if vol_ms:
        t = statistics.mean(vol_ms) * 1e-3
        ach = FLOP_PER_PAIR * nv_local * nc / t / 1e12
        kernels.append({"kernel": "eval_kernel<deform> (volume)", "ms": t * 1e3, "bound": "fp64",
                        "achieved": ach, "peak": peak_tf, "unit": "TFLOP/s", "frac": ach / peak_tf,
                        "traffic": traffic.get("eval_kernel")})
    if sweep_ms:
        kernels.append({"kernel": "rbf_errors_argmax_dev (sharded final sweep, this rank's slice)",
                        "ms": statistics.mean(sweep_ms)})
    if getattr(res.history, "device_mode", None) == "grid":
        # the grid path's appends stream four packed triangles per append (Li for
        # c0 and for c, L for r, the column copy for u): 4 * 8 n(n+1)/2 bytes at n
        # supports; against the measured HBM copy bandwidth (small factors are
        # L2-resident, so this is the algorithmic rate, not DRAM traffic)
        t2 = sum(r.t2_s for r in res.history.records)
        tri_bytes = sum(16.0 * n * (n + 1) for n in range(3, nc))
        hbm = None
        try:
            hbm = json.loads((REPO / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs")
        except (OSError, ValueError):
            pass
        if t2 > 0:
            ach = tri_bytes / t2 / 1e9
            kernels.append({"kernel": "gcb_grid_kernel appends (t2: triangle streams)", "ms": t2 * 1e3,
                            "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                            "frac": ach / hbm if hbm else None,
                            "bytes_per_append": "16 n (n + 1): four packed triangles (SURVEY 8(d): 8 n^2 = two)",
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs" if hbm else "none"})
    dominant = max((k for k in kernels if "frac" in k and k["unit"] == "TFLOP/s"), key=lambda k: k["ms"]) if kernels else None

    cpu = cpu1 = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = host_threads()
        s = cpu_oracle_step(wl, threads, args.cpu_sample)
        cpu = {"value": s["pairs"] / s["seconds"], "unit": UNIT, "cores": threads, "kind": "port",
               "ms_per_step": s["seconds"] * 1e3, "sample": cpu_sample_desc(wl, s, threads),
               "cpu_model": cpu_model()}
        s1 = cpu_oracle_step(wl, 1, args.cpu_sample)
        cpu1 = {"value": s1["pairs"] / s1["seconds"], "unit": UNIT, "cores": 1, "kind": "port",
                "ms_per_step": s1["seconds"] * 1e3, "sample": cpu_sample_desc(wl, s1, 1)}

    if rank == 0:
        h2d = (wl.nb * 48 + wl.nb * 4 + (wl.m + 1) * 4 + nv_local * 24 + nc * 48)
        d2h = (nv_local * 24 + nc * (4 + 24) + 64 + 40 * (len(res.history.records) + 1))
        roof = None
        if dominant:
            roof = {"bound": "fp64", "achieved": dominant["achieved"], "peak": peak_tf,
                    "unit": "TFLOP/s", "frac": dominant["frac"], "traffic": dominant["traffic"],
                    "traffic_source": "profiles/ncu_traffic.json (ncu --set full, per launch)",
                    "kernel": dominant["kernel"], "peak_source": peak["source"],
                    "note": "the selection loop is latency bound (dependent DSMEM hops between "
                            "phases, DESIGN.md 4.2); the volume kernel's roofline is in kernels[]"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_total / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak" if replicas else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, paper_2004_04817_b200/workloads.py)",
            "config": config_desc(wl, world, mode=mode),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / args.steps * 1e3,
                    "host_memory": "volume in pinned host memory; boundary as numpy arrays; "
                                   "partition recomputed every step"},
            "e2e_pageable": {"value": pairs_per_step / e2e_pg, "unit": UNIT, "ms_per_step": e2e_pg * 1e3,
                             "host_memory": "volume as a pageable numpy array (median of "
                                            f"{len(e2e_pageable)} steps)"},
            "roofline": roof,
            "kernels": kernels,
            "fp64_peak": peak,
            "cpu_baseline": cpu,
            "cpu_baseline_1_worker": cpu1,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
            "volume_ms": vol_shard_max,
            "volume_ms_source": "volume kernel alone on this rank's shard, median of 5, max over ranks",
            "breakdown": {"nc": nc, "selection_pairs": a_sel, "volume_pairs": wl.nv * nc,
                          "iterations": len(res.history.records),
                          # the reference's per-stage columns (cli.py:38), device clock:
                          # t1 = error scans, t2 = solves/appends (selection.py:310-371)
                          "t1_ms": 1e3 * sum(r.t1_s for r in res.history.records),
                          "t2_ms": 1e3 * sum(r.t2_s for r in res.history.records),
                          "selection_ms": statistics.mean(sel_ms) if sel_ms else None,
                          "volume_ms": statistics.mean(vol_ms) if vol_ms else None,
                          "converged": bool(res.converged) if res.converged is not None else None,
                          "loop_mode": getattr(res.history, "device_mode", None),
                          "loop_phase_us": {k: v / 1.965e3 for k, v in
                                            getattr(prof_hist, "device_phase_cycles", {}).items()
                                            if k not in ("appends", "iterations")},
                          "loop_phase_source": "one extra untimed selection with the phase clock on",
                          "loop_counts": {k: getattr(prof_hist, "device_phase_cycles", {}).get(k)
                                          for k in ("appends", "iterations")}},
        }
        if vol_full_ms is not None:
            line["volume_ms_1gpu"] = vol_full_ms
            line["volume_speedup"] = vol_full_ms / vol_shard_max
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return relaunch(args)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        return 2
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
