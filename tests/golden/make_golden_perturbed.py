"""The reference's own sequence sensitivity on configs[3] (Nb = 200k, R = 4, m = 64).

Runs the REFERENCE (``/root/reference``) a second time with ONE equally valid change
to its arithmetic: the bordered-Cholesky append's forward substitution
(``CholeskyState.append`` -> ``_forward``, reference core.py:145-151, 171) gets one
step of iterative refinement, ``c += L^-1 (row - L c)``; everything else is the
stock reference. The refined solve is at least as accurate as the stock one, so a
support sequence that is determined by the FP64 problem must not change. The
position where the two reference runs first differ is where the selection stops
being determined by FP64 arithmetic -- a bound on how far ANY implementation (this
repository's GPU loop included) can match the stock reference's sequence.

Writes tests/golden/cfg3_m64_refined.npz: the refined run's sequence, its record
nodes and local maxima, and ``first_difference`` against cfg3_m64.npz.

    python tests/golden/make_golden_perturbed.py       # ~13 CPU minutes (8 workers)
"""

import os
import sys

import numpy as np
from scipy.linalg import solve_triangular

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import make_golden as MG  # noqa: E402
import make_golden_large as ML  # noqa: E402

RC = MG.RC
_stock_append = RC.CholeskyState.append


def refined_append(self, new_row):
    """Stock append, but the cross vector gets one refinement step."""
    new_row = np.asarray(new_row, dtype=float)
    n = self._n
    if n == 0 or new_row.shape != (n + 1,):
        return _stock_append(self, new_row)
    cross = self._forward(new_row[:n])[:n]
    L = self._L[:n, :n]
    cross = cross + solve_triangular(L, new_row[:n] - L @ cross, lower=True, check_finite=False)
    pivot2 = new_row[n] - cross @ cross
    if not pivot2 > 0.0:
        raise RC.NotPositiveDefiniteError(f"pivot^2 = {pivot2:.3e} appending row {n}")
    if n + 1 > self._L.shape[0]:
        grown = np.eye(2 * self._L.shape[0])
        grown[:n, :n] = self._L[:n, :n]
        self._L = grown
    self._L[n, :n] = cross
    self._L[n, n] = np.sqrt(pivot2)
    self._n = n + 1
    return self


def main():
    RC.CholeskyState.append = refined_append
    wl = MG.W.config(3, nv=10)
    out, res = ML.run(wl.points, wl.disp, wl.radius, wl.tol, wl.nb, 64)
    g = np.load(os.path.join(os.path.dirname(__file__), "cfg3_m64.npz"))
    a, b = out["seq"], g["seq"]
    k = min(len(a), len(b))
    diff = np.flatnonzero(a[:k] != b[:k])
    first = int(diff[0]) if len(diff) else (k if len(a) != len(b) else -1)
    print("first difference vs the stock reference:", first, "Nc", len(a), "vs", len(b), flush=True)
    MG.save("cfg3_m64_refined", seq=a, rec_node=out["rec_node"], rec_local_max=out["rec_local_max"],
            weights=out["weights"], first_difference=np.array(first), converged=out["converged"])


if __name__ == "__main__":
    main()
