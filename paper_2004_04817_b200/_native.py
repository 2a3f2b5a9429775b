"""ctypes binding of the sm_100a C ABI declared in ``include/rbf_b200.h``.

There is no CPU fallback: if the shared library or a CUDA device is
missing, every compute call raises :class:`NativeUnavailableError`.
"""

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import NativeUnavailableError

# RBF_LIB: an alternative build of the library (A/B experiments, tools/ab_build.sh)
_LIB_PATH = (Path(os.environ["RBF_LIB"]) if os.environ.get("RBF_LIB")
             else Path(__file__).resolve().parent / "_lib" / "librbf_b200.so")

RBF_OK = 0
RBF_EARG = 1
RBF_ECUDA = 2
RBF_ENOTPD = 3
RBF_ENCCL = 4
RBF_EGROW = 5
RBF_ESTALL = 6
RBF_EPARSE = 7
GCB_PHASES = 1  # rbf_gcb_args.flags: record per-phase SM cycles
GCB_NO_OVERLAP = 2  # rbf_gcb_args.flags: MSG path without the overlapped next-group scan
GCB_NO_TAIL = 4  # rbf_gcb_args.flags: one-cluster final sweep without the whole-GPU tail launch
GCB_NO_SWEEP = 8  # rbf_gcb_args.flags: end the loop without the final sweep (the caller sweeps)
GCB_REFINE = 16  # rbf_gcb_args.flags: MSG path refines every append (default: once min l_i^2 < 1e-7)
STATUS_DONE = 1
GCB_AUTO = 0
GCB_CLUSTER = 1
GCB_GRID = 2
GCB_SMEM = 3
GCB_MSG = 4

c_dp = ctypes.c_void_p  # device pointers are passed as integers


class GcbRecord(ctypes.Structure):
    _fields_ = [
        ("group", ctypes.c_int32),
        ("node_pos", ctypes.c_int32),
        ("added", ctypes.c_int32),
        ("n_before", ctypes.c_int32),
        ("local_max", ctypes.c_double),
        ("t1_s", ctypes.c_double),
        ("t2_s", ctypes.c_double),
    ]


RECORD_DTYPE = np.dtype(
    [("group", "<i4"), ("node_pos", "<i4"), ("added", "<i4"), ("n_before", "<i4"),
     ("local_max", "<f8"), ("t1_s", "<f8"), ("t2_s", "<f8")]
)
assert RECORD_DTYPE.itemsize == ctypes.sizeof(GcbRecord) == 40


class GcbState(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("streak_ok", ctypes.c_int32),
        ("streak_noadd", ctypes.c_int32),
        ("n_records", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("fail_row", ctypes.c_int32),
        ("done_loop", ctypes.c_int32),
        ("fail_pivot2", ctypes.c_double),
        ("t2_carry", ctypes.c_double),
        ("final_max", ctypes.c_double),
        ("final_pos", ctypes.c_int32),
        ("fault", ctypes.c_int32),
        ("want_mode", ctypes.c_int32),
        ("handover", ctypes.c_int32),
        ("phase_cycles", ctypes.c_double * 16),
    ]


assert ctypes.sizeof(GcbState) == 200
PHASES = ["scan", "fold_row", "c0", "r", "c", "pivot_cols", "bookkeeping", "seeds", "final_sweep",
          "appends", "iterations", "scan_compute", "scan_reduce", "scan_epilogue", "scan_partials",
          "cols_partials"]


class GcbArgs(ctypes.Structure):
    _fields_ = [
        ("points", c_dp),
        ("disp", c_dp),
        ("group_pos", c_dp),
        ("group_off", c_dp),
        ("nb", ctypes.c_int32),
        ("m", ctypes.c_int32),
        ("mode", ctypes.c_int32),
        ("max_supports", ctypes.c_int32),
        ("clusters", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("radius", ctypes.c_double),
        ("tol", ctypes.c_double),
        ("dup_dist", ctypes.c_double),
        ("L", c_dp),
        ("Li", c_dp),
        ("y", c_dp),
        ("sup", c_dp),
        ("sel", c_dp),
        ("inel", c_dp),
        ("cap", ctypes.c_int32),
        ("records", c_dp),
        ("rec_cap", ctypes.c_int32),
        ("state", c_dp),
        ("scratch", c_dp),
        ("scratch_bytes", ctypes.c_size_t),
    ]


# (name, restype, argtypes) for every symbol include/rbf_b200.h declares
SIGNATURES = [
    ("rbf_abi_version", ctypes.c_int, []),
    ("rbf_last_error", ctypes.c_char_p, []),
    ("rbf_device_info", ctypes.c_int,
     [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]),
    ("rbf_eval", ctypes.c_int,
     [c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, c_dp, c_dp]),
    ("rbf_eval_loop", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    ("rbf_eval_host_loop", ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                          ctypes.c_void_p, ctypes.c_double, ctypes.c_int, ctypes.c_void_p,
                                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    ("rbf_eval_host", ctypes.c_int,
     [c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_int64, ctypes.c_double, ctypes.c_int, c_dp, c_dp, c_dp,
      ctypes.c_int, c_dp]),
    ("rbf_errors_scratch_bytes", ctypes.c_size_t, [ctypes.c_int64]),
    ("rbf_errors_argmax", ctypes.c_int,
     [c_dp, c_dp, c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_int64, ctypes.c_double, c_dp,
      ctypes.POINTER(ctypes.c_double), c_dp, ctypes.c_size_t, c_dp]),
    ("rbf_errors_argmax_dev", ctypes.c_int,
     [c_dp, c_dp, c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_int64, ctypes.c_double, c_dp,
      ctypes.c_int64, c_dp, c_dp, ctypes.c_size_t, c_dp]),
    ("rbf_best_fold", ctypes.c_int, [c_dp, ctypes.c_int64, c_dp, c_dp]),
    ("rbf_nearest", ctypes.c_int, [c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, c_dp, c_dp]),
    ("rbf_chol_scratch_bytes", ctypes.c_size_t, [ctypes.c_int64]),
    ("rbf_chol_points_scratch_bytes", ctypes.c_size_t, [ctypes.c_int64]),
    ("rbf_chol_append_points", ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                              ctypes.c_void_p, ctypes.c_double, ctypes.POINTER(ctypes.c_int64),
                                              ctypes.POINTER(ctypes.c_double), ctypes.c_void_p, ctypes.c_size_t,
                                              ctypes.c_void_p]),
    ("rbf_chol_append", ctypes.c_int,
     [c_dp, c_dp, ctypes.c_int64, c_dp, ctypes.POINTER(ctypes.c_double), c_dp, ctypes.c_size_t, c_dp]),
    ("rbf_chol_solve", ctypes.c_int,
     [c_dp, c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, c_dp, c_dp, ctypes.c_size_t, c_dp]),
    ("rbf_gcb_ctas", ctypes.c_int,
     [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
      ctypes.POINTER(ctypes.c_int32)]),
    ("rbf_gcb_scratch_bytes", ctypes.c_size_t, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]),
    ("rbf_gcb_run", ctypes.c_int, [ctypes.POINTER(GcbArgs), c_dp]),
    ("rbf_partition", ctypes.c_int,
     [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
      ctypes.c_int64, c_dp, c_dp]),
    ("rbf_l2_release", ctypes.c_int, []),
    ("rbf_mdk1_counts", ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]),
    ("rbf_mdk1_parse", ctypes.c_int,
     [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, c_dp, c_dp, c_dp,
      ctypes.c_int]),
    ("rbf_disp_parse", ctypes.c_int, [ctypes.c_char_p, ctypes.c_size_t, c_dp, ctypes.c_int64, c_dp, ctypes.c_int]),
    ("rbf_mdk1_format_nodes", ctypes.c_int64, [c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, ctypes.c_int]),
    ("rbf_disp_format", ctypes.c_int64, [c_dp, c_dp, ctypes.c_int64, c_dp, ctypes.c_int64, ctypes.c_int]),
    ("rbf_fp64_probe_scratch_bytes", ctypes.c_size_t, [ctypes.c_int]),
    ("rbf_fp64_probe", ctypes.c_int, [ctypes.c_int, c_dp, ctypes.POINTER(ctypes.c_double), c_dp]),
]

_lib = None


def lib_path():
    return _LIB_PATH


def load(build_if_missing=True):
    """Load (building first if needed) the shared library. Does not need a GPU."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists() and build_if_missing:
        from . import _build

        _build.build()
    if not _LIB_PATH.exists():
        raise NativeUnavailableError(f"native library missing: {_LIB_PATH}")
    lib = ctypes.CDLL(os.fspath(_LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.rbf_abi_version() != 1:
        raise NativeUnavailableError("ABI version mismatch")
    _lib = lib
    return lib


def last_error():
    return (load().rbf_last_error() or b"").decode(errors="replace")


def check(rc, what):
    """Map a non-OK return code to the package's exception classes."""
    if rc == RBF_OK:
        return
    from . import errors as E

    msg = f"{what}: {last_error()}"
    if rc == RBF_ENOTPD:
        raise E.NotPositiveDefiniteError(last_error())
    if rc == RBF_EARG:
        raise ValueError(msg)
    if rc == RBF_ESTALL:
        raise E.SelectionStalledError(msg)
    raise NativeUnavailableError(msg)


_torch = None


def torch():
    """torch, for device buffers and streams (plumbing only)."""
    global _torch
    if _torch is None:
        import torch as _t

        _torch = _t
    return _torch


def require_cuda():
    """Fail loudly (no CPU fallback) unless a CUDA device and the library exist."""
    t = torch()
    if not t.cuda.is_available():
        raise NativeUnavailableError(
            "paper_2004_04817_b200 needs a CUDA (sm_100a) device; no CPU fallback exists"
        )
    return load()


def stream_ptr(stream=None):
    t = torch()
    s = stream if stream is not None else t.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dptr(tensor):
    return ctypes.c_void_p(tensor.data_ptr())


# ------------------------------------------------------ launch accounting
class LaunchLog:
    """Counts this library's kernel launches and (optionally) brackets them
    with CUDA events on the launching stream, for bench.py's per-kernel
    timings and its ``gpu_launches`` figure."""

    def __init__(self, timing=False):
        self.timing = timing
        self.count = 0
        self.by_name = {}
        self.spans = []  # (name, start_event, end_event)

    def kernel_ms(self, name):
        torch().cuda.synchronize()
        return [a.elapsed_time(b) for n, a, b in self.spans if n == name]


_log = None


class launch_log:
    def __init__(self, timing=False):
        self.log = LaunchLog(timing)

    def __enter__(self):
        global _log
        self._prev = _log
        _log = self.log
        return self.log

    def __exit__(self, *exc):
        global _log
        _log = self._prev
        return False


class launching:
    """``with launching("rbf_eval", kernels=1): rc = lib.rbf_eval(...)``"""

    def __init__(self, name, kernels=1):
        self.name = name
        self.kernels = kernels

    def __enter__(self):
        log = _log
        if log is not None:
            log.count += self.kernels
            log.by_name[self.name] = log.by_name.get(self.name, 0) + self.kernels
            if log.timing:
                t = torch()
                self.e0 = t.cuda.Event(enable_timing=True)
                self.e1 = t.cuda.Event(enable_timing=True)
                self.e0.record()
        return self

    def __exit__(self, *exc):
        log = _log
        if log is not None and log.timing:
            self.e1.record()
            log.spans.append((self.name, self.e0, self.e1))
        return False
