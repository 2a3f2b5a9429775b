"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain numpy/scipy restatement of the reference ``rbfdeform`` hot path
(arXiv 2004.04817, GCB-greedy RBF mesh deformation), used as the parity
checker by ``tests/``, by ``__graft_entry__.smoke()`` and as the
``cpu_baseline`` / ``--impl reference`` arm of ``bench.py``. The product
package ``paper_2004_04817_b200`` never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks this restatement bit for
bit against golden vectors that ``tests/golden/make_golden.py`` produced by
running the reference itself (``/root/reference/pkg/src/rbfdeform``) on the
same inputs, and -- when the reference is importable -- directly against
the reference on fresh seeded inputs.

Third-party arithmetic: the reference leaves the floating-point work to
scipy ``cdist`` (C++), numpy ufuncs and OpenBLAS (dgemm, dtrsm via LAPACK
dtrtrs); this restatement calls the very same routines in the same order
with the same operand shapes, so on one machine it reproduces the
reference's bits. Only minimum versions are pinned upstream
(pyproject.toml:10-15: numpy>=1.24, scipy>=1.10); goldens were produced
with numpy 2.3.5 / scipy 1.18.1 / scipy-openblas 0.3.30.
"""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.linalg import solve_triangular
from scipy.spatial.distance import cdist
from threadpoolctl import threadpool_limits

# reference core.py:26, 31, 35 and selection.py:43
ROWS_PER_SPAN = 2048
COLS_PER_TILE = 512
SOLVE_PAD = 256
DUP_FRACTION = 1e-12


def phi(eta):
    """Wendland C2, separately rounded chain (reference core.py:45-50)."""
    t = np.maximum(1.0 - eta, 0.0)
    t *= t
    t *= t
    return t * (4.0 * eta + 1.0)


def _padded_supports(targets, sup_pts, sup_w, radius):
    """Zero-weight sentinels beyond every target up to a tile multiple
    (reference core.py:284-298)."""
    k = len(sup_pts)
    extra = -k % COLS_PER_TILE
    if extra == 0:
        return sup_pts, sup_w
    far = max(float(np.abs(sup_pts).max()) if k else 0.0,
              float(np.abs(targets).max()) if len(targets) else 0.0, 1.0)
    sentinel = np.full((extra, 3), far + 2.0 * radius)
    return np.vstack([sup_pts, sentinel]), np.vstack([sup_w, np.zeros((extra, 3))])


def eval_sum(targets, sup_pts, sup_w, radius, threads=1):
    """out[k] = sum_i w_i phi(|p_k - s_i| / R), span x tile blocked
    (reference core.py:301-334)."""
    targets = np.asarray(targets, dtype=float)
    n = len(targets)
    out = np.zeros((n, 3))
    sp, sw = _padded_supports(targets, np.asarray(sup_pts, float), np.asarray(sup_w, float), radius)

    def span(lo):
        hi = min(lo + ROWS_PER_SPAN, n)
        block = targets[lo:hi]
        for c in range(0, len(sp), COLS_PER_TILE):
            d = cdist(block, sp[c : c + COLS_PER_TILE])
            d /= radius
            t = np.maximum(1.0 - d, 0.0)
            t *= t
            t *= t
            d *= 4.0
            d += 1.0
            t *= d
            out[lo:hi] += t @ sw[c : c + COLS_PER_TILE]

    starts = list(range(0, n, ROWS_PER_SPAN))
    with threadpool_limits(limits=1, user_api="blas"):
        if threads > 1 and len(starts) > 1:
            with ThreadPoolExecutor(max_workers=threads) as pool:
                list(pool.map(span, starts))
        else:
            for lo in starts:
                span(lo)
    return out


def residual_errors(positions, pts, disp, sup_pts, sup_w, radius, threads=1):
    """|disp - interpolant| per boundary row (reference selection.py:215-221)."""
    pred = eval_sum(pts[positions], sup_pts, sup_w, radius, threads)
    r = disp[positions] - pred
    return np.sqrt((r * r).sum(axis=1))


def argmax_low(errors, ids):
    """Row of the max, exact ties to the smallest id (selection.py:231-234)."""
    rows = np.flatnonzero(errors == errors.max())
    return int(rows[np.argmin(ids[rows])])


class Factor:
    """Growing Cholesky factor in a capacity buffer with unit trailing
    diagonal; substitutions run on 256-row-rounded sizes
    (reference core.py:115-205)."""

    def __init__(self):
        self.buf = np.eye(8)
        self.n = 0

    def _size(self):
        cap = len(self.buf)
        if cap <= SOLVE_PAD:
            return cap
        return min(-(-self.n // SOLVE_PAD) * SOLVE_PAD, cap)

    def _lower_solve(self, rhs):
        s = self._size()
        b = np.zeros((s,) + rhs.shape[1:])
        b[: self.n] = rhs
        return solve_triangular(self.buf[:s, :s], b, lower=True, check_finite=False)

    def try_append(self, row):
        """Returns pivot^2; appends only when pivot^2 > 0 (core.py:153-185)."""
        n = self.n
        if n == 0:
            c, p2 = np.empty(0), row[0]
        else:
            c = self._lower_solve(row[:n])[:n]
            p2 = row[n] - c @ c
        if not p2 > 0.0:
            return p2
        if n + 1 > len(self.buf):
            bigger = np.eye(2 * len(self.buf))
            bigger[:n, :n] = self.buf[:n, :n]
            self.buf = bigger
        self.buf[n, :n] = c
        self.buf[n, n] = np.sqrt(p2)
        self.n = n + 1
        return p2

    def solve(self, rhs):
        """(L L^T) x = rhs (core.py:187-205)."""
        if self.n == 0:
            return rhs.copy()
        y = self._lower_solve(rhs)
        s = len(y)
        x = solve_triangular(self.buf[:s, :s], y, lower=True, trans="T", check_finite=False)
        return x[: self.n]

    @property
    def L(self):
        return self.buf[: self.n, : self.n].copy()


def partition(nb, m, seed):
    """PCG64 permutation dealt round-robin, groups unsorted (selection.py:177-185)."""
    perm = np.random.default_rng(seed).permutation(nb)
    return [perm[j::m] for j in range(m)]


def seeds(pts, disp):
    """argmax |d|, then two farthest-point picks (selection.py:198-212)."""
    chosen = [int(np.argmax(np.linalg.norm(disp, axis=1)))]
    dmin = np.linalg.norm(pts - pts[chosen[0]], axis=1)
    for _ in range(2):
        nxt = int(np.argmax(dmin))
        chosen.append(nxt)
        dmin = np.minimum(dmin, np.linalg.norm(pts - pts[nxt], axis=1))
    return chosen


def select(pts, disp, radius, tol, max_supports, m=1, seed=0, threads=1, ids=None):
    """The GCB / greedy loop (reference selection.py:274-421).

    Returns a dict: ``seq`` selected positions in order, ``weights`` (Nc, 3),
    ``records`` (iteration, group, node_pos, local_max, kernel_evals) per
    visit, ``final`` (iteration, node_pos, global_max, kernel_evals),
    ``converged``. Raises RuntimeError('stalled') / ArithmeticError('notpd')
    where the reference raises SelectionStalledError / NotPositiveDefiniteError.
    """
    pts = np.asarray(pts, float)
    disp = np.asarray(disp, float)
    nb = len(pts)
    ids = np.arange(nb) if ids is None else np.asarray(ids)
    groups = partition(nb, m, seed)
    fac = Factor()
    chosen = []
    blocked = np.zeros(nb, dtype=bool)
    with threadpool_limits(limits=1, user_api="blas"):
        for p in seeds(pts, disp):
            d = cdist(pts[p][None, :], pts[chosen])[0] if chosen else np.empty(0)
            p2 = fac.try_append(np.append(phi(d / radius), 1.0))
            if not p2 > 0.0:
                raise ArithmeticError(f"notpd {p2} row {fac.n}")
            chosen.append(p)
            blocked[p] = True
        sup = pts[chosen]
        records = []
        w = None
        stale = True
        evals_total = 0
        ok_run = 0
        idle_run = 0
        it = 3
        while len(chosen) < max_supports:
            if stale:
                w = fac.solve(disp[chosen])
                stale = False
            g = it % m
            rows = groups[g]
            err = residual_errors(rows, pts, disp, sup, w, radius, threads)
            evals = len(rows) * len(chosen)
            evals_total += evals
            top = argmax_low(err, ids[rows])
            peak = float(err[top])
            took = None
            if peak > tol:
                for r in np.lexsort((ids[rows], -err)):
                    if err[r] <= tol:
                        break
                    p = int(rows[r])
                    if blocked[p]:
                        continue
                    d = cdist(pts[p][None, :], sup)[0]
                    if d.min() < DUP_FRACTION * radius:
                        blocked[p] = True
                        continue
                    if not fac.try_append(np.append(phi(d / radius), 1.0)) > 0.0:
                        blocked[p] = True
                        continue
                    chosen.append(p)
                    blocked[p] = True
                    sup = pts[chosen]
                    took = p
                    stale = True
                    break
            records.append((it, g, took if took is not None else int(rows[top]), peak, evals))
            if took is None:
                idle_run += 1
                ok_run = ok_run + 1 if peak <= tol else 0
                if ok_run >= m:
                    break
                if idle_run >= m:
                    raise RuntimeError("stalled")
            else:
                idle_run = ok_run = 0
            it += 1
        if stale:
            w = fac.solve(disp[chosen])
        err = residual_errors(np.arange(nb), pts, disp, sup, w, radius, threads)
        worst = argmax_low(err, ids)
        final = (it + 1, worst, float(err[worst]), nb * len(chosen))
    return {
        "seq": np.array(chosen, dtype=np.int64),
        "weights": w,
        "records": records,
        "final": final,
        "converged": final[2] <= tol,
        "L": fac.L,
    }


# ------------------------------------------------------------------ metrics
KL_FLOOR = 1e-12  # reference metrics.py:14-16


def nearest_distances(pts, sup_pts):
    """min over supports of cdist (reference metrics.py:45-48)."""
    return cdist(pts, sup_pts).min(axis=1)


def kl_divergence(pts, sup1, sup2):
    """reference metrics.py:63-74"""
    d1 = nearest_distances(pts, sup1)
    d2 = np.maximum(nearest_distances(pts, sup2), KL_FLOOR)
    mask = d1 > 0.0
    return float(np.sum(d1[mask] * np.log(d1[mask] / d2[mask])))


def error_summary(pts, disp, ids, sup_pts, sup_w, radius):
    """(max, rms, id of max) over all boundary rows (reference metrics.py:77-88)."""
    errors = residual_errors(np.arange(len(pts)), pts, disp, sup_pts, sup_w, radius)
    worst = argmax_low(errors, ids)
    return float(errors[worst]), float(np.sqrt(np.mean(errors * errors))), int(ids[worst])


def error_history(pts, disp, ids, support_ids, radius, every=50):
    """Per-prefix summaries with a one-shot Cholesky per prefix
    (reference metrics.py:91-115)."""
    from scipy.linalg import cho_factor, cho_solve

    support_ids = np.asarray(support_ids, dtype=np.intp)
    total = len(support_ids)
    counts = list(range(every, total, every))
    if not counts or counts[-1] != total:
        counts.append(total)
    positions = np.searchsorted(ids, support_ids)
    out = []
    with threadpool_limits(1):
        for n in counts:
            p = pts[positions[:n]]
            a = phi(cdist(p, p) / radius)
            w = cho_solve(cho_factor(a, lower=True), disp[positions[:n]])
            out.append((n, error_summary(pts, disp, ids, p, w, radius)))
    return out


def default_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1
