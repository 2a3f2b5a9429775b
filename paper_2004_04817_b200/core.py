"""RBF core on the B200: kernel helpers, the device-resident growing Cholesky
factor and the volume evaluation.

Drop-in mirror of reference ``core.py`` (same names, arguments, return
types and exceptions). The cheap host helpers ``wendland_c2``,
``normalized_distance``, ``kernel_matrix`` and ``assemble_phi``
(reference core.py:53-112) stay numpy, as in the reference; everything on
the hot path (``_eval_displacements`` core.py:301-334, ``CholeskyState``
core.py:115-205) runs in the sm_100a library through the C ABI of
``include/rbf_b200.h``. No CPU fallback: without a CUDA device the
compute entry points raise ``NativeUnavailableError``.

``workers`` is accepted for signature compatibility and ignored: results
never depended on it in the reference (core.py:24-26) and do not here.
"""

from dataclasses import dataclass

import numpy as np
from scipy.spatial.distance import cdist

from . import _native as N
from .errors import (
    DimensionMismatchError,
    DuplicateNodesError,
    EmptySupportSetError,
    NotPositiveDefiniteError,
)


# --------------------------------------------------------------- host helpers
def _phi(eta):
    """Wendland C2 on nonnegative eta (reference core.py:45-50)."""
    t = np.maximum(1.0 - eta, 0.0)
    t *= t
    t *= t
    return t * (4.0 * eta + 1.0)


def wendland_c2(eta):
    """(1 - eta)^4 (4 eta + 1) for eta <= 1, else 0 (reference core.py:53-70)."""
    eta = np.asarray(eta, dtype=float)
    if np.isnan(eta).any():
        raise ValueError("eta must not contain NaN")
    if (eta < 0).any():
        raise ValueError("eta must be nonnegative")
    out = _phi(eta)
    return float(out) if out.ndim == 0 else out


def normalized_distance(a, b, radius):
    """Euclidean distance divided by the radius (reference core.py:73-79)."""
    if radius <= 0:
        raise ValueError(f"radius must be positive, got {radius}")
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / radius)


def kernel_matrix(points_a, points_b, radius):
    """phi(|a_i - b_j| / R), shape (len(a), len(b)) (reference core.py:82-88)."""
    if radius <= 0:
        raise ValueError(f"radius must be positive, got {radius}")
    return _phi(cdist(np.asarray(points_a, float), np.asarray(points_b, float)) / radius)


def assemble_phi(points, radius):
    """Symmetric kernel matrix with unit diagonal (reference core.py:91-112)."""
    if radius <= 0:
        raise ValueError(f"radius must be positive, got {radius}")
    points = np.atleast_2d(np.asarray(points, dtype=float))
    dist = cdist(points, points)
    n = len(points)
    if n > 1:
        masked = dist + np.diag(np.full(n, np.inf))
        i, j = np.unravel_index(np.argmin(masked), dist.shape)
        if masked[i, j] == 0.0:
            raise DuplicateNodesError(f"points {min(i, j)} and {max(i, j)} coincide")
    upper = np.triu(_phi(dist / radius), 1)
    phi = upper + upper.T
    np.fill_diagonal(phi, 1.0)
    return phi


# ------------------------------------------------------------ device helpers
def _device():
    t = N.torch()
    return t.device("cuda", t.cuda.current_device())


def _to_device(a, dtype=None):
    """numpy / torch -> contiguous device tensor (float64 unless dtype)."""
    t = N.torch()
    dtype = dtype or t.float64
    if isinstance(a, t.Tensor):
        return a.to(device=_device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    return t.from_numpy(arr).to(device=_device(), dtype=dtype, non_blocking=True)


def _to_host(tensor):
    """Device tensor -> numpy (through pinned memory for large results)."""
    t = N.torch()
    if tensor.numel() * tensor.element_size() >= (1 << 20):
        host = t.empty(tensor.shape, dtype=tensor.dtype, pin_memory=True)
        host.copy_(tensor, non_blocking=True)
        t.cuda.current_stream().synchronize()
        return host.numpy()
    return tensor.cpu().numpy()


def _tri(n):
    return n * (n + 1) // 2


# ---------------------------------------------------------- Cholesky factor
class CholeskyState:
    """Growing lower-triangular Cholesky factor, device resident.

    Mirrors reference core.py:115-205: ``append`` adds the next row of the
    SPD matrix in O(order^2) and raises :class:`NotPositiveDefiniteError`
    (state unchanged) on a non-positive pivot; ``solve`` solves
    ``(L L^T) x = rhs``; ``order`` and ``factor`` as in the reference.
    Storage: the factor and its inverse as packed lower triangles in HBM
    (capacity doubles like the reference's buffer, core.py:178-181).
    """

    def __init__(self):
        self._n = 0
        self._cap = 0
        self._L = None
        self._Li = None

    @property
    def order(self):
        return self._n

    @property
    def factor(self):
        """Copy of the current (order, order) lower-triangular factor."""
        n = self._n
        out = np.zeros((n, n))
        if n:
            packed = self._L[: _tri(n)].cpu().numpy()
            rows, cols = np.tril_indices(n)
            out[rows, cols] = packed
        return out

    def _reserve(self, n):
        if n <= self._cap:
            return
        t = N.torch()
        cap = max(8, self._cap)
        while cap < n:
            cap *= 2
        L = t.zeros(_tri(cap), dtype=t.float64, device=_device())
        Li = t.zeros(_tri(cap), dtype=t.float64, device=_device())
        if self._n:
            L[: _tri(self._n)] = self._L[: _tri(self._n)]
            Li[: _tri(self._n)] = self._Li[: _tri(self._n)]
        self._L, self._Li, self._cap = L, Li, cap

    def append(self, new_row):
        new_row = np.asarray(new_row, dtype=float)
        n = self._n
        if new_row.shape != (n + 1,):
            raise DimensionMismatchError(f"expected row of length {n + 1}, got shape {new_row.shape}")
        lib = N.require_cuda()
        t = N.torch()
        self._reserve(n + 1)
        row = _to_device(new_row)
        nbytes = lib.rbf_chol_scratch_bytes(n + 1)
        scratch = t.empty(nbytes, dtype=t.uint8, device=_device())
        piv = N.ctypes.c_double(0.0)
        with N.launching("rbf_chol_append", kernels=6 if n else 2):
            rc = lib.rbf_chol_append(N.dptr(self._L), N.dptr(self._Li), n, N.dptr(row),
                                     N.ctypes.byref(piv), N.dptr(scratch), nbytes, N.stream_ptr())
        if rc == N.RBF_ENOTPD:
            raise NotPositiveDefiniteError(
                f"pivot^2 = {piv.value:.3e} appending row {n}; "
                "support nodes may coincide or be nearly coincident"
            )
        N.check(rc, "rbf_chol_append")
        self._n = n + 1
        return self

    def _append_points(self, points, radius):
        """Append the kernel rows of supports ``points[order:]`` against every
        support before them (``points[:order]`` must be the supports already
        factored), built on the device with the reference's kernel_matrix
        rounding, in ONE device pass with no host round trip between rows
        (rbf_chol_append_points). Raises NotPositiveDefiniteError at the first
        non-positive pivot, with the rows before it kept."""
        points = np.ascontiguousarray(points, dtype=float).reshape(-1, 3)
        n0, total = self._n, len(points)
        if total < n0:
            raise DimensionMismatchError(f"{total} points for a factor of order {n0}")
        if total == n0:
            return self
        lib = N.require_cuda()
        t = N.torch()
        self._reserve(total)
        sup = _to_device(points)
        nbytes = lib.rbf_chol_points_scratch_bytes(total + 1)
        scratch = t.empty(nbytes, dtype=t.uint8, device=_device())
        done = N.ctypes.c_int64(0)
        piv = N.ctypes.c_double(0.0)
        with N.launching("rbf_chol_append_points", kernels=7 * (total - n0)):
            rc = lib.rbf_chol_append_points(N.dptr(self._L), N.dptr(self._Li), n0, total - n0, N.dptr(sup),
                                            float(radius), N.ctypes.byref(done), N.ctypes.byref(piv),
                                            N.dptr(scratch), nbytes, N.stream_ptr())
        if rc == N.RBF_ENOTPD:
            self._n = n0 + int(done.value)
            raise NotPositiveDefiniteError(
                f"pivot^2 = {piv.value:.3e} appending row {self._n}; "
                "support nodes may coincide or be nearly coincident"
            )
        N.check(rc, "rbf_chol_append_points")
        self._n = total
        return self

    def solve(self, rhs):
        rhs = np.asarray(rhs, dtype=float)
        if rhs.shape[:1] != (self._n,):
            raise DimensionMismatchError(
                f"rhs has leading dimension {rhs.shape[:1]}, factor order is {self._n}"
            )
        return self._solve_prefix(rhs, self._n)

    def _solve_prefix(self, rhs, n):
        """Solve with the leading order-n block of the factor (the factor of
        the first n appended rows; a prefix of the packed triangles)."""
        rhs = np.asarray(rhs, dtype=float)
        if not 0 <= n <= self._n or rhs.shape[:1] != (n,):
            raise DimensionMismatchError(f"prefix {n} / rhs {rhs.shape} vs factor order {self._n}")
        if n == 0:
            return rhs.copy()
        lib = N.require_cuda()
        t = N.torch()
        k = 1 if rhs.ndim == 1 else int(np.prod(rhs.shape[1:]))
        b = _to_device(rhs.reshape(n, k))
        out = t.empty_like(b)
        nbytes = 3 * n * k * 8
        scratch = t.empty(nbytes, dtype=t.uint8, device=_device())
        with N.launching("rbf_chol_solve", kernels=6 * ((k + 3) // 4)):
            rc = lib.rbf_chol_solve(N.dptr(self._L), N.dptr(self._Li), n, N.dptr(b), k,
                                    N.dptr(out), N.dptr(scratch), nbytes, N.stream_ptr())
        N.check(rc, "rbf_chol_solve")
        return _to_host(out).reshape(rhs.shape)


def cholesky_append(state, new_row):
    """Functional spelling of :meth:`CholeskyState.append` (core.py:208-210)."""
    return state.append(new_row)


def solve_weights(state, displacements):
    """(order, 3) weights for (order, 3) displacements (core.py:213-224)."""
    displacements = np.asarray(displacements, dtype=float)
    if displacements.ndim != 2 or displacements.shape[1] != 3:
        raise DimensionMismatchError(f"displacements must be (order, 3), got {displacements.shape}")
    return state.solve(displacements)


@dataclass(eq=False)
class SupportSet:
    """Selected support nodes with their weights (reference core.py:227-265)."""

    nodes: np.ndarray
    points: np.ndarray
    weights: np.ndarray

    def __post_init__(self):
        self.nodes = np.asarray(self.nodes, dtype=np.intp)
        self.points = np.asarray(self.points, dtype=float)
        self.weights = np.asarray(self.weights, dtype=float)
        n = len(self.nodes)
        if len(np.unique(self.nodes)) != n:
            raise ValueError("support node ids must be unique")
        if self.points.shape != (n, 3) or self.weights.shape != (n, 3):
            raise DimensionMismatchError(
                f"points {self.points.shape} and weights {self.weights.shape} must both be ({n}, 3)"
            )

    def __len__(self):
        return len(self.nodes)

    @property
    def wx(self):
        return self.weights[:, 0]

    @property
    def wy(self):
        return self.weights[:, 1]

    @property
    def wz(self):
        return self.weights[:, 2]


def solve_support_weights(points, displacements, radius):
    """Factor the kernel matrix of ``points`` row by row and solve for
    (n, 3) weights (reference core.py:268-281)."""
    points = np.asarray(points, dtype=float)
    displacements = np.asarray(displacements, dtype=float)
    state = CholeskyState()
    state._append_points(points, radius)  # the rows of the loop above, in one device pass
    return solve_weights(state, displacements)


# --------------------------------------------------------------- evaluation
def eval_device(points, support_points, weights, radius, deform=False, out=None):
    """Device-resident evaluation: torch tensors in, torch tensor out.

    ``points`` (n, 3), ``support_points`` / ``weights`` (Nc, 3) float64
    CUDA tensors. Returns U (or points + U when ``deform``).
    """
    lib = N.require_cuda()
    t = N.torch()
    n = points.shape[0]
    if out is None:
        out = t.empty((n, 3), dtype=t.float64, device=points.device)
    with N.launching("rbf_eval", kernels=1 if n else 0):
        rc = lib.rbf_eval(N.dptr(points), n, N.dptr(support_points), N.dptr(weights),
                          support_points.shape[0], float(radius), 1 if deform else 0,
                          N.dptr(out), N.stream_ptr())
    N.check(rc, "rbf_eval")
    return out


_PIPELINE_MIN = 1 << 18   # host inputs at least this long are streamed in chunks
_PIPELINE_CHUNKS = 8


def _eval_host_pipelined(points, s, w, radius, deform):
    """Host (n, 3) points -> host result through the library's chunked
    copy / kernel / copy pipeline (rbf_eval_host): the host->device copy of
    chunk k+1 and the device->host copy of chunk k-1 overlap the kernel on
    chunk k. Per-target results are bitwise those of one launch."""
    lib = N.require_cuda()
    t = N.torch()
    n = len(points)
    src = t.from_numpy(points)  # pinned memory copies asynchronously; pageable ones are staged
    dev_in = t.empty((n, 3), dtype=t.float64, device=_device())
    dev_out = t.empty((n, 3), dtype=t.float64, device=_device())
    host_out = t.empty((n, 3), dtype=t.float64, pin_memory=True)
    with N.launching("rbf_eval", kernels=_PIPELINE_CHUNKS):
        rc = lib.rbf_eval_host(src.data_ptr(), n, N.dptr(s), N.dptr(w), s.shape[0], float(radius),
                               1 if deform else 0, N.dptr(dev_in), N.dptr(dev_out), host_out.data_ptr(),
                               _PIPELINE_CHUNKS, N.stream_ptr())
    N.check(rc, "rbf_eval_host")
    t.cuda.current_stream().synchronize()
    return host_out.numpy()


def _eval_displacements(points, support_points, weights, radius, workers=1, deform=False):
    """sum_i w_i phi(|p - s_i| / R) at every point (reference core.py:301-334)."""
    t = N.torch()
    N.require_cuda()
    as_torch = isinstance(points, t.Tensor)
    n = len(points)
    if n == 0:
        return t.zeros((0, 3), dtype=t.float64) if as_torch else np.zeros((0, 3))
    s = _to_device(support_points)
    w = _to_device(weights)
    if not as_torch and n >= _PIPELINE_MIN:
        return _eval_host_pipelined(np.ascontiguousarray(points, dtype=np.float64), s, w, radius, deform)
    p = _to_device(points)
    out = eval_device(p, s, w, radius, deform=deform)
    return out if as_torch else _to_host(out)


def evaluate_displacements(points, support, radius, workers=1):
    """Interpolated displacements, shape (n, 3) (reference core.py:337-351).

    numpy in -> numpy out; a CUDA tensor in -> CUDA tensor out.
    """
    if radius <= 0:
        raise ValueError(f"radius must be positive, got {radius}")
    if len(support) == 0:
        raise EmptySupportSetError("support set is empty")
    t = N.torch()
    if not isinstance(points, t.Tensor):
        points = np.asarray(points, dtype=float).reshape(-1, 3)
    return _eval_displacements(points, support.points, support.weights, radius, workers)


def evaluate_displacement(p, support, radius):
    """Interpolated displacement at one point, shape (3,) (core.py:354-356)."""
    return evaluate_displacements(np.asarray(p, dtype=float)[None, :], support, radius)[0]


def deform_points(points, support, radius, workers=1):
    """``points`` shifted by their interpolated displacements
    (reference core.py:359-367); the add is fused into the kernel epilogue."""
    t = N.torch()
    if isinstance(points, t.Tensor):
        if points.shape[0] == 0:
            return points.clone()
        if radius <= 0:
            raise ValueError(f"radius must be positive, got {radius}")
        if len(support) == 0:
            raise EmptySupportSetError("support set is empty")
        return _eval_displacements(points, support.points, support.weights, radius, deform=True)
    points = np.asarray(points, dtype=float).reshape(-1, 3)
    if len(points) == 0:
        return points.copy()
    if radius <= 0:
        raise ValueError(f"radius must be positive, got {radius}")
    if len(support) == 0:
        raise EmptySupportSetError("support set is empty")
    return _eval_displacements(points, support.points, support.weights, radius, deform=True)
