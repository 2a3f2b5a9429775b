"""Support-node selection (greedy and grouped-circular greedy) on the B200.

Drop-in mirror of reference ``selection.py``. The data types stay numpy;
the seeded PCG64 partition (selection.py:177-185) is computed on the host
by the library's restatement of numpy's PCG64 permutation (bit-identical,
``rbf_partition``) and cached per (Nb, m, seed); the whole selection loop
(``_gcb_run``, selection.py:274-421, seeds selection.py:198-212 included)
runs as ONE persistent kernel of the sm_100a library (``rbf_gcb_run``,
csrc/rbf_gcb.cu). The host reads the support set, weights and
per-iteration records back once, at the end.

Timings in the records come from the device clock (%globaltimer) around
the same stages the reference brackets with ``perf_counter``: t1 = group
scan, t2 = weights update + candidate appends (carried into the next
record, selection.py:310-316, 357).
"""

import os
import threading
from collections import OrderedDict
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native as N
from .core import (
    SupportSet,
    _device,
    _to_device,
    _to_host,
    _tri,
    evaluate_displacement,
    solve_support_weights,
)
from .errors import (
    EmptyGroupError,
    InvalidCountError,
    InvalidGroupCountError,
    NotPositiveDefiniteError,
    SelectionStalledError,
    TooFewBoundaryNodesError,
    UnknownIndexError,
)

# reference selection.py:43
NEAR_DUPLICATE_FRACTION = 1e-12


@dataclass(eq=False)
class BoundarySet:
    """Boundary nodes with prescribed displacements (selection.py:46-83)."""

    indices: np.ndarray
    points: np.ndarray
    disp: np.ndarray

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.intp)
        self.points = np.asarray(self.points, dtype=float)
        self.disp = np.asarray(self.disp, dtype=float)
        nb = len(self.indices)
        if nb == 0:
            raise ValueError("boundary set is empty")
        if self.points.shape != (nb, 3) or self.disp.shape != (nb, 3):
            raise ValueError(
                f"points {self.points.shape} and disp {self.disp.shape} must both be ({nb}, 3)"
            )
        if nb > 1 and not (np.diff(self.indices) > 0).all():
            raise ValueError("boundary indices must be strictly increasing")
        if not np.isfinite(self.points).all() or not np.isfinite(self.disp).all():
            raise ValueError("boundary points and displacements must be finite")

    def __len__(self):
        return len(self.indices)

    def position_of(self, index):
        pos = int(np.searchsorted(self.indices, index))
        if pos == len(self.indices) or self.indices[pos] != index:
            raise UnknownIndexError(f"{index} is not a boundary node")
        return pos


@dataclass(eq=False)
class GroupPartition:
    """m disjoint balanced groups of boundary ids (selection.py:86-102)."""

    m: int
    groups: list
    seed: int

    def __post_init__(self):
        sizes = [len(g) for g in self.groups]
        if len(self.groups) != self.m or min(sizes) < 1:
            raise InvalidGroupCountError("partition must have m nonempty groups")
        if max(sizes) - min(sizes) > 1:
            raise InvalidGroupCountError("group sizes must differ by at most 1")
        merged = np.concatenate(self.groups)
        if len(np.unique(merged)) != len(merged):
            raise InvalidGroupCountError("groups must be disjoint")


@dataclass(frozen=True)
class SelectionConfig:
    """Selection knobs (selection.py:105-126). ``workers`` is accepted and
    ignored: the device path has one result for any worker count."""

    radius: float
    tol: float
    max_supports: int
    m: int = 1
    seed: int = 0
    workers: int = 1

    def __post_init__(self):
        if self.radius <= 0:
            raise ValueError(f"radius must be positive, got {self.radius}")
        if self.tol <= 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_supports < 3:
            raise ValueError(f"max_supports must be >= 3, got {self.max_supports}")
        if self.m < 1:
            raise InvalidGroupCountError(f"m must be >= 1, got {self.m}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")


@dataclass(frozen=True)
class IterationRecord:
    iteration: int
    group: int
    node: int
    local_max_error: float
    kernel_evals: int
    cum_kernel_evals: int
    t1_s: float
    t2_s: float


@dataclass(eq=False)
class SelectionHistory:
    records: list = field(default_factory=list)
    seed: int = 0
    m: int = 1
    final_sweep: IterationRecord | None = None
    t3_s: float | None = None


@dataclass(eq=False)
class SelectionResult:
    support: SupportSet
    history: SelectionHistory
    converged: bool


@dataclass
class KernelEvalCounter:
    count: int = 0

    def add(self, n):
        self.count += int(n)


class _RecordList(list):
    """``SelectionHistory.records`` as a real list whose IterationRecord
    objects are built from the device's record columns on first use (building
    a few hundred frozen dataclasses costs ~0.4 ms; most callers never look).
    Every list operation materialises first, so it behaves as a plain list."""

    __slots__ = ("_cols",)

    def __init__(self, cols):
        super().__init__()
        self._cols = cols

    def _load(self):
        cols = self._cols
        if cols is not None:
            self._cols = None
            list.extend(self, [IterationRecord(*v) for v in zip(*cols)])
        return self

    def __len__(self):
        cols = self._cols
        return len(cols[0]) if cols is not None else list.__len__(self)

    def __bool__(self):
        return len(self) > 0

    def __repr__(self):
        return list.__repr__(self._load())

    def __reduce__(self):
        return (list, (list(self._load()),))


def _lazy(name):
    base = getattr(list, name)

    def method(self, *a, **k):
        return base(self._load(), *a, **k)

    method.__name__ = name
    return method


for _name in ("__getitem__", "__iter__", "__reversed__", "__contains__", "__eq__", "__ne__",
              "__lt__", "__le__", "__gt__", "__ge__", "__add__", "__iadd__", "__mul__", "__imul__",
              "__rmul__", "__setitem__", "__delitem__", "append", "extend", "insert", "pop",
              "remove", "index", "count", "sort", "reverse", "copy", "clear"):
    setattr(_RecordList, _name, _lazy(_name))


# ------------------------------------------------------------ host-side logic
def _partition_native(nb, m, seed):
    """Group positions and offsets from the library's host restatement of
    numpy's PCG64 permutation (rbf_partition): same bits, ~3x faster than
    numpy's shuffle plus the slicing. Returns (flat int32, off int32)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = st["state"], st["inc"]
    mask = (1 << 64) - 1
    flat = np.empty(nb, dtype=np.int32)
    off = np.empty(m + 1, dtype=np.int32)
    lib = N.load()
    N.check(lib.rbf_partition(s >> 64, s & mask, inc >> 64, inc & mask, nb, m,
                              flat.ctypes.data, off.ctypes.data), "rbf_partition")
    return flat, off


def _partition_positions(nb, m, seed):
    """PCG64 permutation dealt round-robin (selection.py:183-184); returns the
    permutation, the groups' positions concatenated (group j = perm[j::m])
    and the m+1 offsets."""
    perm = np.random.default_rng(seed).permutation(nb)
    q = -(-nb // m)
    padded = np.full(q * m, -1, dtype=np.int64)
    padded[:nb] = perm
    flat = padded.reshape(q, m).T.ravel()
    flat = flat[flat >= 0]
    sizes = np.full(m, nb // m, dtype=np.int64)
    sizes[: nb % m] += 1
    off = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(sizes, out=off[1:])
    return perm, flat, off


def stage_boundary(boundary):
    """Keep device copies of ``boundary.points`` / ``.disp`` on the current
    GPU so repeated selections start from HBM-resident inputs (the arrays
    must not be modified afterwards; re-stage if they are)."""
    boundary._device = (boundary.points, boundary.disp, _to_device(boundary.points),
                        _to_device(boundary.disp))
    return boundary


# Reuse across selections (thread-safe): the partition depends only on
# (nb, m, seed), so its device copy is cached; loop buffers hold no user data
# once a selection has returned (results are host copies), so they go back to
# a pool keyed by shape and device. A selection takes its buffers out of the
# pool for its whole run: concurrent selections never share them.
_cache_lock = threading.Lock()
_part_cache = OrderedDict()  # (device, nb, m, seed) -> (off, gpos, goff)
_PART_CACHE_MAX = 16
_buf_pool = {}               # (device, nb, cap, rec_cap, ctas) -> [_LoopBuffers]


_part_pool = None  # one worker: the host shuffle runs beside the caller's device set-up


def _drop_part_pool():
    global _part_pool
    _part_pool = None  # a forked child has no worker thread: it makes its own pool


if hasattr(os, "register_at_fork"):
    os.register_at_fork(after_in_child=_drop_part_pool)


def _partition_device_start(nb, m, seed):
    """Start the partition for (nb, m, seed); returns a callable that yields
    (off, gpos, goff) with the device copies made on the caller's stream. On
    a cache miss the PCG64 shuffle (a native call that releases the GIL, ~0.2
    ms for 20k nodes) runs on a worker thread while the caller uploads the
    boundary and prepares the loop buffers."""
    global _part_pool
    t = N.torch()
    key = (t.cuda.current_device(), nb, m, seed)
    with _cache_lock:
        hit = _part_cache.get(key)
        if hit is not None:
            _part_cache.move_to_end(key)
            return lambda: hit
        if _part_pool is None:
            from concurrent.futures import ThreadPoolExecutor

            _part_pool = ThreadPoolExecutor(max_workers=1, thread_name_prefix="rbf-partition")
    fut = _part_pool.submit(_partition_native, nb, m, seed)

    def finish():
        flat, off = fut.result()
        part = (off, _to_device(flat, dtype=t.int32), _to_device(off, dtype=t.int32))
        with _cache_lock:
            _part_cache[key] = part
            while len(_part_cache) > _PART_CACHE_MAX:
                _part_cache.popitem(last=False)
        return part

    return finish


def _partition_device(nb, m, seed):
    return _partition_device_start(nb, m, seed)()


def _take_buffers(nb, cap, rec_cap, ctas):
    key = (N.torch().cuda.current_device(), nb, cap, rec_cap, ctas)
    with _cache_lock:
        free = _buf_pool.get(key)
        buf = free.pop() if free else None
    if buf is None:
        return key, _LoopBuffers(nb, cap, rec_cap, ctas)
    busy = getattr(buf, "busy", None)
    if busy is not None:  # a kernel queued by read_all(then) may still read the buffers
        N.torch().cuda.current_stream().wait_event(busy)
        buf.busy = None
    buf.reset()
    return key, buf


def _give_buffers(key, buf):
    with _cache_lock:
        free = _buf_pool.setdefault(key, [])
        if len(free) < 2:
            free.append(buf)


def _boundary_on_device(boundary):
    cached = getattr(boundary, "_device", None)
    if cached is not None and cached[0] is boundary.points and cached[1] is boundary.disp:
        return cached[2], cached[3]
    return _to_device(boundary.points), _to_device(boundary.disp)


def partition_boundary(boundary, m, seed):
    """Seeded balanced partition of the boundary ids (selection.py:177-185)."""
    nb = len(boundary)
    if not 1 <= m <= nb:
        raise InvalidGroupCountError(f"m must be in [1, {nb}], got {m}")
    perm = np.random.default_rng(seed).permutation(nb)
    groups = [boundary.indices[perm[j::m]] for j in range(m)]
    return GroupPartition(m=m, groups=groups, seed=seed)


def seed_supports(boundary):
    """Initial support triple (selection.py:188-195)."""
    return boundary.indices[_seed_positions(boundary)]


def _seed_positions(boundary):
    """Largest |disp| first, then two farthest-point picks; first
    occurrence wins ties (selection.py:198-212)."""
    if len(boundary) < 3:
        raise TooFewBoundaryNodesError(f"need at least 3 boundary nodes, got {len(boundary)}")
    mags = np.linalg.norm(boundary.disp, axis=1)
    chosen = [int(np.argmax(mags))]
    dmin = np.linalg.norm(boundary.points - boundary.points[chosen[0]], axis=1)
    for _ in range(2):
        nxt = int(np.argmax(dmin))
        chosen.append(nxt)
        dmin = np.minimum(dmin, np.linalg.norm(boundary.points - boundary.points[nxt], axis=1))
    return chosen


def _argmax_lowest_id(errors, ids):
    """Row of the maximum, ties to the smallest id (selection.py:231-234)."""
    best = np.flatnonzero(errors == errors.max())
    return int(best[np.argmin(ids[best])])


# ------------------------------------------------------------ device scans
def _errors_device(positions, boundary, support_points, weights, radius, want_errors=True):
    """Fused device error scan + (err, lowest position) arg-max. The boundary
    is uploaded per call unless it was staged (``stage_boundary``: then the
    HBM copy is used and a per-group caller moves only the group's positions)."""
    lib = N.require_cuda()
    t = N.torch()
    pts, disp = _boundary_on_device(boundary)
    pos = _to_device(np.asarray(positions, dtype=np.int64), dtype=t.int64)
    sp = _to_device(support_points)
    w = _to_device(weights)
    n = len(positions)
    err = t.empty(n, dtype=t.float64, device=_device()) if want_errors else None
    nbytes = lib.rbf_errors_scratch_bytes(n)
    scratch = t.empty(nbytes, dtype=t.uint8, device=_device())
    best = (N.ctypes.c_double * 2)()
    with N.launching("rbf_errors_argmax", kernels=3):
        rc = lib.rbf_errors_argmax(N.dptr(pts), N.dptr(disp), N.dptr(pos), n, N.dptr(sp), N.dptr(w),
                                   sp.shape[0], float(radius), N.dptr(err) if err is not None else None,
                                   best, N.dptr(scratch), nbytes, N.stream_ptr())
    N.check(rc, "rbf_errors_argmax")
    errors = _to_host(err) if err is not None else None
    return errors, float(best[0]), int(best[1])


def _errors_at(positions, boundary, support_points, weights, radius, workers=1):
    """|disp - interpolant| at boundary rows (selection.py:215-221)."""
    positions = np.asarray(positions, dtype=np.int64)
    if len(positions) == 0:
        return np.zeros(0)
    errors, _, _ = _errors_device(positions, boundary, support_points, weights, radius)
    return errors


def interpolation_error(index, boundary, support, radius):
    """Residual norm at one boundary node (selection.py:224-228)."""
    pos = boundary.position_of(index)
    predicted = evaluate_displacement(boundary.points[pos], support, radius)
    return float(np.linalg.norm(boundary.disp[pos] - predicted))


def group_arg_max_error(group, boundary, support, radius, counter=None):
    """(node id, error) of the worst node in ``group`` (selection.py:237-254),
    one fused device scan + arg-max."""
    group = np.asarray(group, dtype=np.intp)
    if len(group) == 0:
        raise EmptyGroupError("group is empty")
    positions = np.searchsorted(boundary.indices, group)
    _, err, pos = _errors_device(positions, boundary, support.points, support.weights, radius,
                                 want_errors=False)
    if counter is not None:
        counter.add(len(group) * len(support))
    return int(boundary.indices[pos]), err


# --------------------------------------------------------------- the loop
class _LoopBuffers:
    """Device buffers of one selection run; grown on RBF_EGROW."""

    def __init__(self, nb, cap, rec_cap, ctas):
        t = N.torch()
        dev = _device()
        self.t = t
        self.dev = dev
        self.nb = nb
        self.ctas = ctas
        self.cap = 0
        self.rec_cap = 0
        self.L = self.Li = self.y = self.sup = self.sel = None
        self.records = None
        self.inel = t.zeros(nb, dtype=t.uint8, device=dev)
        self.state = t.zeros(N.ctypes.sizeof(N.GcbState), dtype=t.uint8, device=dev)
        self._grow_factor(cap, 0)
        self._grow_records(rec_cap, 0)

    def reset(self):
        """Fresh run state on reused buffers (the kernel starts from n = 0)."""
        self.inel.zero_()
        self.state.zero_()

    def _grow_factor(self, cap, n):
        t, dev = self.t, self.dev
        # every row is written by the kernel before it is read: no zero fill
        L = t.empty(_tri(cap), dtype=t.float64, device=dev)
        Li = t.empty(_tri(cap), dtype=t.float64, device=dev)
        y = t.empty((cap, 3), dtype=t.float64, device=dev)
        # SoA: x, y, z, wx, wy, wz, then the compensated weights' hi (3) and lo (3) rows
        sup = t.empty((12, cap), dtype=t.float64, device=dev)
        sel = t.empty(cap, dtype=t.int32, device=dev)
        if n:
            L[: _tri(n)] = self.L[: _tri(n)]
            Li[: _tri(n)] = self.Li[: _tri(n)]
            y[:n] = self.y[:n]
            sup[:, :n] = self.sup[:, :n]
            sel[:n] = self.sel[:n]
        self.L, self.Li, self.y, self.sup, self.sel, self.cap = L, Li, y, sup, sel, cap
        lib = N.load()
        self.scratch_bytes = lib.rbf_gcb_scratch_bytes(self.nb, cap, self.ctas)
        self.scratch = t.empty(self.scratch_bytes, dtype=t.uint8, device=dev)

    def _staging(self):
        sz = N.ctypes.sizeof(N.GcbState) + self.cap * 4 + 3 * self.cap * 8 + self.records.numel()
        if getattr(self, "_host", None) is None or self._host.numel() < sz:
            self._host = self.t.empty(sz, dtype=self.t.uint8, pin_memory=True)
        return self._host

    def read_all(self, then=None):
        """Async copies of state, sel, weight rows and records into one
        pinned buffer, one synchronisation; returns (state, host bytes).
        ``then(self)`` is queued on the stream behind the copies (the host
        waits for the copies only, not for it)."""
        t = self.t
        host = self._staging()
        ss = N.ctypes.sizeof(N.GcbState)
        o1 = ss
        o2 = o1 + self.cap * 4
        o3 = o2 + 3 * self.cap * 8
        o4 = o3 + self.records.numel()
        host[:o1].copy_(self.state, non_blocking=True)
        host[o1:o2].copy_(self.sel.view(t.uint8), non_blocking=True)
        host[o2:o3].copy_(self.sup[3:6].reshape(-1).view(t.uint8), non_blocking=True)
        host[o3:o4].copy_(self.records.reshape(-1), non_blocking=True)
        copied = t.cuda.Event()
        copied.record()
        self.then_queued = False
        if then is not None:  # queued behind the copies: runs while the host unpacks
            self.then_queued = bool(then(self))
            self.busy = t.cuda.Event()
            self.busy.record()
        copied.synchronize()
        hb = host.numpy()
        self._offsets = (o1, o2, o3)
        return N.GcbState.from_buffer_copy(hb[:ss].tobytes()), hb

    def unpack(self, hb, n, nrec):
        o1, o2, o3 = self._offsets
        sel = hb[o1:o1 + 4 * n].view(np.int32).astype(np.intp)
        w = hb[o2:o2 + 24 * self.cap].view(np.float64).reshape(3, self.cap)[:, :n]
        weights = np.ascontiguousarray(w.T)
        recs = hb[o3:o3 + nrec * N.RECORD_DTYPE.itemsize].view(N.RECORD_DTYPE).copy()
        return sel, weights, recs

    def resize_scratch(self, ctas):
        self.ctas = ctas
        lib = N.load()
        self.scratch_bytes = lib.rbf_gcb_scratch_bytes(self.nb, self.cap, ctas)
        self.scratch = self.t.empty(self.scratch_bytes, dtype=self.t.uint8, device=self.dev)

    def _grow_records(self, rec_cap, nrec):
        t = self.t
        rec = t.empty((rec_cap, N.RECORD_DTYPE.itemsize), dtype=t.uint8, device=self.dev)
        if nrec:
            rec[:nrec] = self.records[:nrec]
        self.records, self.rec_cap = rec, rec_cap


def _read_state(buf):
    raw = buf.state.cpu().numpy().tobytes()
    return N.GcbState.from_buffer_copy(raw)




def _initial_capacity(config, nb):
    limit = min(config.max_supports, nb) + 1
    return int(max(8, min(limit, 1024)))


def gcb_select(boundary, config):
    """Grouped-circular greedy selection (selection.py:257-271); the loop of
    selection.py:274-421 runs on the device."""
    return _gcb_run(boundary, config)


def _gcb_run(boundary, config, mode=None, phases=None, sweep=True, then=None):
    """The device loop. ``sweep=False`` stops before the final sweep
    (RBF_GCB_NO_SWEEP; multi.gcb_select shards it over ranks): the returned
    history's ``final_sweep`` then carries the iteration number, counters and
    t2 but ``node`` = -1 and a NaN maximum, and ``converged`` is None."""
    nb = len(boundary)
    m = config.m
    if not 1 <= m <= nb:
        raise InvalidGroupCountError(f"m must be in [1, {nb}], got {m}")
    if nb < 3:
        raise TooFewBoundaryNodesError(f"need at least 3 boundary nodes, got {nb}")
    radius = float(config.radius)
    lib = N.require_cuda()
    t = N.torch()
    partition = _partition_device_start(nb, m, config.seed)  # joined below, after the device set-up

    ctas = N.ctypes.c_int32(0)
    resolved = N.ctypes.c_int32(0)
    if mode is None:  # RBF_GCB_MODE=msg|smem|cluster|grid overrides the automatic choice
        import os

        name = os.environ.get("RBF_GCB_MODE", "").lower()
        mode = {"msg": N.GCB_MSG, "smem": N.GCB_SMEM, "cluster": N.GCB_CLUSTER,
                "grid": N.GCB_GRID}.get(name)
    want = N.GCB_AUTO if mode is None else mode
    N.check(lib.rbf_gcb_ctas(want, nb, m, N.ctypes.byref(ctas), N.ctypes.byref(resolved)),
            "rbf_gcb_ctas")
    pts, disp = _boundary_on_device(boundary)
    cap = _initial_capacity(config, nb)
    bkey, buf = _take_buffers(nb, cap, 2 * cap + m + 8, ctas.value)

    args = N.GcbArgs()
    args.points, args.disp = pts.data_ptr(), disp.data_ptr()
    try:
        off, gpos, goff = partition()
    except BaseException:
        _give_buffers(bkey, buf)
        raise
    args.group_pos, args.group_off = gpos.data_ptr(), goff.data_ptr()
    args.nb, args.m = nb, m
    args.mode = resolved.value
    args.max_supports = int(min(config.max_supports, 2**31 - 1))
    import os

    args.clusters = int(os.environ.get("RBF_GCB_CLUSTERS", "0"))
    if phases is None:  # RBF_GCB_PHASES=1: per-phase device cycles in history.device_phase_cycles
        phases = os.environ.get("RBF_GCB_PHASES", "") == "1"
    args.flags = N.GCB_PHASES if phases else 0
    if os.environ.get("RBF_GCB_OVERLAP", "1") == "0":  # A/B: no next-group scan during appends
        args.flags |= N.GCB_NO_OVERLAP
    if os.environ.get("RBF_GCB_TAIL", "1") == "0":  # A/B: final sweep inside the one-cluster launch
        args.flags |= N.GCB_NO_TAIL
    if os.environ.get("RBF_GCB_REFINE", "") == "1":  # A/B: MSG appends always refined
        args.flags |= N.GCB_REFINE
    if not sweep:
        args.flags |= N.GCB_NO_SWEEP
    args.radius = radius
    args.tol = float(config.tol)
    args.dup_dist = NEAR_DUPLICATE_FRACTION * config.radius
    stream = N.stream_ptr()
    limit = min(config.max_supports, nb) + 1
    used_grid = False
    while True:
        args.L, args.Li, args.y = buf.L.data_ptr(), buf.Li.data_ptr(), buf.y.data_ptr()
        args.sup, args.sel, args.inel = buf.sup.data_ptr(), buf.sel.data_ptr(), buf.inel.data_ptr()
        args.cap = buf.cap
        args.records, args.rec_cap = buf.records.data_ptr(), buf.rec_cap
        args.state = buf.state.data_ptr()
        args.scratch, args.scratch_bytes = buf.scratch.data_ptr(), buf.scratch_bytes
        used_grid = used_grid or args.mode == N.GCB_GRID
        # one-cluster shapes queue a whole-GPU tail launch for the final sweep
        # (twice when runs within tolerance go to the tail: m >= 16)
        tail = args.mode in (N.GCB_MSG, N.GCB_SMEM) and not (args.flags & N.GCB_NO_TAIL)
        with N.launching("rbf_gcb_run", kernels=(4 if m >= 16 else 2) if tail else 1):
            rc = lib.rbf_gcb_run(N.ctypes.byref(args), stream)
        N.check(rc, "rbf_gcb_run")
        # state, selection, weights and records in one staged read (the kernel
        # is stream-ordered before the copies): one synchronisation per launch
        st, host = buf.read_all(None if then is None else (lambda b, mode=args.mode: then(b, mode)))
        then_done = buf.then_queued and st.status == N.STATUS_DONE
        if st.status == N.STATUS_DONE:
            break
        if st.status == N.RBF_ENOTPD:
            raise NotPositiveDefiniteError(
                f"pivot^2 = {st.fail_pivot2:.3e} appending row {st.fail_row}; "
                "support nodes may coincide or be nearly coincident"
            )
        if st.status == N.RBF_ESTALL:
            raise SelectionStalledError(
                "errors above tolerance remain but no group has an addable candidate"
            )
        if st.status != N.RBF_EGROW:
            raise N.NativeUnavailableError(f"selection kernel ended with status {st.status}")
        if st.want_mode != args.mode:
            # the shared-memory path is full: resume in the L2-resident path
            N.check(lib.rbf_gcb_ctas(st.want_mode, nb, m, N.ctypes.byref(ctas),
                                     N.ctypes.byref(resolved)), "rbf_gcb_ctas")
            args.mode = resolved.value
            buf.resize_scratch(ctas.value)
            continue
        if st.n >= buf.cap:
            buf._grow_factor(max(min(2 * buf.cap, limit), st.n + 1), st.n)
        if st.n_records >= buf.rec_cap:
            buf._grow_records(2 * buf.rec_cap, st.n_records)

    if used_grid:
        N.check(lib.rbf_l2_release(), "rbf_l2_release")
    n = st.n
    nrec = st.n_records
    sel, weights, recs = buf.unpack(host, n, nrec)
    _give_buffers(bkey, buf)  # (a scratch sized for more CTAs also serves fewer)

    sizes = np.diff(off)
    history = SelectionHistory(seed=config.seed, m=m)
    idx = boundary.indices
    body = recs[:-1] if sweep else recs
    groups = body["group"].astype(np.int64)
    evals = sizes[groups] * body["n_before"].astype(np.int64)
    cum = np.cumsum(evals)
    nodes = idx[body["node_pos"]]
    history.records = _RecordList((
        range(3, 3 + len(body)), groups.tolist(), nodes.tolist(), body["local_max"].tolist(),
        evals.tolist(), cum.tolist(), body["t1_s"].tolist(), body["t2_s"].tolist()))
    sweep_evals = nb * n
    total = (int(cum[-1]) if len(cum) else 0) + sweep_evals
    if sweep:
        fin = recs[-1]
        history.final_sweep = IterationRecord(
            iteration=st.k + 1,
            group=-1,
            node=int(idx[fin["node_pos"]]),
            local_max_error=float(fin["local_max"]),
            kernel_evals=sweep_evals,
            cum_kernel_evals=total,
            t1_s=float(fin["t1_s"]),
            t2_s=float(fin["t2_s"]),
        )
    else:  # the caller sweeps (multi.gcb_select)
        history.final_sweep = IterationRecord(
            iteration=st.k + 1, group=-1, node=-1, local_max_error=float("nan"),
            kernel_evals=sweep_evals, cum_kernel_evals=total, t1_s=0.0, t2_s=float(st.t2_carry))
    # diagnostics: SM cycles of CTA 0 per phase of the device loop
    history.device_phase_cycles = dict(zip(N.PHASES, list(st.phase_cycles))) if phases else {}
    history.device_mode = {N.GCB_CLUSTER: "cluster", N.GCB_GRID: "grid", N.GCB_SMEM: "smem",
                           N.GCB_MSG: "msg"}[args.mode]
    support = SupportSet(nodes=idx[sel], points=boundary.points[sel], weights=weights)
    result = SelectionResult(
        support=support, history=history,
        converged=(float(fin["local_max"]) <= config.tol) if sweep else None,
    )
    if then is not None:
        result._then_done = then_done  # the queued follow-up ran on the final state
    return result


def select_and_deform(boundary, config, points, out=None):
    """gcb_select followed by deform_points of ``points`` over the selected
    support set, as one device sequence (the reference's cmd_deform,
    cli.py:158-182, and RBFMeshDeformer's fit + transform): the volume work is
    queued on the selection's stream right behind the loop, reading the
    supports, weights and their count from the loop's own buffers on the
    device, so it runs while the host reads back and unpacks the selection.

    * ``points`` a CUDA tensor (n, 3): one volume kernel (rbf_eval_loop);
      ``out`` (or a new tensor) receives the moved points in stream order.
    * ``points`` host (n, 3) array: copied to the device on a side stream while
      the loop runs (pageable arrays staged through pinned memory piece by
      piece), then chunked kernels + result copies (rbf_eval_host_loop) into
      a pinned host result -- when the loop runs in a one-cluster shape (it
      then finishes in the same call); otherwise the two calls one after the
      other.

    Returns (SelectionResult, moved). Bitwise the values of the two calls."""
    from .core import _PIPELINE_CHUNKS, _device, deform_points

    t = N.torch()
    if config.radius <= 0:
        raise ValueError(f"radius must be positive, got {config.radius}")
    lib = N.require_cuda()
    on_device = isinstance(points, t.Tensor) and points.is_cuda
    if on_device:
        pts = points.reshape(-1, 3)
        if pts.dtype != t.float64 or not pts.is_contiguous():
            pts = pts.to(t.float64).contiguous()
        if out is None:
            out = t.empty_like(pts)
    else:
        host = np.ascontiguousarray(np.asarray(points, dtype=np.float64).reshape(-1, 3))
        pts = t.from_numpy(host)
        dev_in = t.empty(pts.shape, dtype=t.float64, device=_device())
        dev_out = t.empty_like(dev_in)
        out = t.empty(pts.shape, dtype=t.float64, pin_memory=True)
    n = pts.shape[0]
    if n == 0:
        res = gcb_select(boundary, config)
        return res, (out if on_device else out.numpy())

    uploaded = [None]

    def upload():
        """The volume to the device on a side stream while the loop runs (a
        concurrent 48 MB copy slows the one-cluster loop by ~1 %,
        tools/dma_interference.py); a pageable array is staged into pinned
        memory by the host in pieces, each piece's copy issued as soon as it is
        staged. Once per call; the fallback below reuses the copy."""
        if uploaded[0] is not None:
            return
        side = t.cuda.Stream()
        if pts.is_pinned():
            with t.cuda.stream(side):
                dev_in.copy_(pts, non_blocking=True)
        else:
            staged = t.empty(pts.shape, dtype=t.float64, pin_memory=True)
            step = max(1, -(-n // 4))
            for lo in range(0, n, step):
                staged[lo:lo + step].copy_(pts[lo:lo + step])
                with t.cuda.stream(side):
                    dev_in[lo:lo + step].copy_(staged[lo:lo + step], non_blocking=True)
            uploaded.append(staged)  # keep the staging buffer alive until the copies ran
        ev = t.cuda.Event()
        ev.record(side)
        uploaded[0] = ev

    # the result copies of a round that does not finish the loop are wasted
    # (and the caller's stream waits for them): queue the pipeline in a
    # one-cluster round only for groups of up to ~1,000 nodes (card * 383 <=
    # 4e5 pairs) -- configs[0-1], whose runs end within the one-cluster
    # capacity of 383 supports; larger groups (configs[2]) reach the capacity
    # and move on to the grid
    card_max = -(-len(boundary) // config.m)
    queue_pipeline = card_max * 383 <= 400_000

    def then(buf, mode):
        if on_device:
            with N.launching("rbf_eval", kernels=1):
                rc = lib.rbf_eval_loop(N.dptr(pts), n, buf.sup.data_ptr(), buf.cap, buf.state.data_ptr(),
                                       float(config.radius), 1, N.dptr(out), N.stream_ptr())
            N.check(rc, "rbf_eval_loop")
            return True
        upload()
        if mode not in (N.GCB_MSG, N.GCB_SMEM) or not queue_pipeline:
            return False  # this round may not finish the loop: no result copies yet
        t.cuda.current_stream().wait_event(uploaded[0])
        with N.launching("rbf_eval", kernels=_PIPELINE_CHUNKS):
            rc = lib.rbf_eval_host_loop(None, n, buf.sup.data_ptr(), buf.cap, buf.state.data_ptr(),
                                        float(config.radius), 1, N.dptr(dev_in), N.dptr(dev_out),
                                        out.data_ptr(), _PIPELINE_CHUNKS, N.stream_ptr())
        N.check(rc, "rbf_eval_host_loop")
        return True

    try:
        res = _gcb_run(boundary, config, then=then)
    except BaseException:
        t.cuda.synchronize()  # copies queued on the side stream still read our buffers
        raise
    if not getattr(res, "_then_done", False):  # the loop finished in a round without it
        if on_device:
            from .core import eval_device

            sp = t.from_numpy(np.ascontiguousarray(res.support.points)).to(pts.device)
            sw = t.from_numpy(np.ascontiguousarray(res.support.weights)).to(pts.device)
            eval_device(pts, sp, sw, config.radius, deform=True, out=out)
            return res, out
        if uploaded[0] is None:
            return res, deform_points(host, res.support, config.radius)
        # the volume is on the device already: kernels + result copies only
        t.cuda.current_stream().wait_event(uploaded[0])
        sp = t.from_numpy(np.ascontiguousarray(res.support.points)).to(dev_in.device)
        sw = t.from_numpy(np.ascontiguousarray(res.support.weights)).to(dev_in.device)
        with N.launching("rbf_eval", kernels=_PIPELINE_CHUNKS):
            rc = lib.rbf_eval_host(None, n, N.dptr(sp), N.dptr(sw), sp.shape[0], float(config.radius), 1,
                                   N.dptr(dev_in), N.dptr(dev_out), out.data_ptr(), _PIPELINE_CHUNKS,
                                   N.stream_ptr())
        N.check(rc, "rbf_eval_host")
        t.cuda.current_stream().synchronize()
        return res, out.numpy()
    if on_device:
        return res, out
    t.cuda.current_stream().synchronize()
    return res, out.numpy()


def greedy_select(boundary, config):
    """Traditional greedy: gcb with m = 1 (selection.py:424-428)."""
    return gcb_select(boundary, replace(config, m=1))


def random_select(boundary, n, seed, radius):
    """n seeded uniform ids with solved weights (selection.py:431-442)."""
    nb = len(boundary)
    if not 3 <= n <= nb:
        raise InvalidCountError(f"n must be in [3, {nb}], got {n}")
    positions = np.random.default_rng(seed).choice(nb, size=n, replace=False)
    points = boundary.points[positions]
    weights = solve_support_weights(points, boundary.disp[positions], radius)
    return SupportSet(nodes=boundary.indices[positions], points=points, weights=weights)


def error_stage_cost(history):
    """Error-stage kernel evaluations, final sweep excluded (selection.py:445-448)."""
    return sum(r.kernel_evals for r in history.records)


def resolve_auto_m(boundary, radius, tol, seed=0, workers=1, probe_cap=200):
    """Group count from a short greedy probe (reference cli.py:69-99,
    ``--m auto``): greedy selection to the earlier of ``probe_cap`` supports
    or the tolerance; if it did not converge, the final support count is
    extrapolated from the log-error decay over the second half of the probe;
    returns round(1.5 * Nb / Nc_hat) clipped to [1, Nb] (the middle of the
    recommended [Nb/Nc, 2 Nb/Nc] band). The probe runs on the device."""
    nb = len(boundary)
    cap = min(probe_cap, nb)
    probe = greedy_select(boundary, SelectionConfig(radius=radius, tol=tol, max_supports=max(cap, 3),
                                                    seed=seed, workers=workers))
    n_probe = len(probe.support)
    if probe.converged:
        n_hat = n_probe
    else:
        # m = 1 adds a node at every over-tolerance visit: record r holds 3 + r supports
        err = np.array([r.local_max_error for r in probe.history.records])
        count = 3.0 + np.arange(len(err))
        half = slice(len(err) // 2, None)
        slope, icpt = np.polyfit(count[half], np.log(np.maximum(err[half], 1e-300)), 1)
        n_hat = nb if slope >= 0 else (np.log(tol) - icpt) / slope
        n_hat = min(max(n_hat, n_probe), nb)
    return int(np.clip(round(1.5 * nb / n_hat), 1, nb))
