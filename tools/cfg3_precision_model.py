"""numpy model of the device loop's factor arithmetic on the configs[3] sequence.

Appends the reference's own support sequence (tests/golden/cfg3_m64.npz, first K
supports) three ways and compares the weights and the scan errors of the group where
the device sequence first left the reference's (tools/cfg3_divergence.py: position
4125, group 29):

  ref    the reference's arithmetic (oracle Factor: substitutions, weights solved
         from scratch -- bit-identical to the reference);
  inc    the device loop's scheme: inverse factor Li, c = c0 + Li (row - L c0),
         weights updated incrementally x' = x - (u / l) y_n, u = Li^T c;
  fresh  the same factor, weights recomputed as Li^T y every append;
  refw   incremental weights plus one step of back-substitution refinement,
         x += Li^T (y - L^T x), at the end.

    python tools/cfg3_precision_model.py [K]
"""

import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))


def main():
    import rbf_oracle as O
    from paper_2004_04817_b200 import workloads as W

    K = int(sys.argv[1]) if len(sys.argv) > 1 else 4125
    g = dict(np.load(REPO / "tests/golden/cfg3_m64.npz"))
    wl = W.config(3, nv=10)
    R = wl.radius
    seq = g["seq"][:K]
    P, D = wl.points[seq], wl.disp[seq]
    # reference arithmetic
    F = O.Factor()
    Li = np.zeros((K, K))
    L = np.zeros((K, K))
    y = np.zeros((K, 3))
    x = np.zeros((K, 3))
    xk = np.zeros((K, 3))   # compensated (two-sum) incremental weights
    xk_lo = np.zeros((K, 3))
    xp = np.zeros((K, 3))   # fresh every PERIOD appends, incremental between
    PERIOD = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    for n in range(K):
        d = np.sqrt(((P[:n] - P[n]) ** 2).sum(1)) if n else np.zeros(0)
        row = np.append(O.phi(d / R), 1.0)
        assert F.try_append(row) > 0
        # device scheme
        if n == 0:
            l = 1.0
            c = np.zeros(0)
        else:
            c0 = Li[:n, :n] @ row[:n]
            r = row[:n] - L[:n, :n] @ c0
            c = c0 + Li[:n, :n] @ r
            l = np.sqrt(1.0 - c @ c)
        yn = (D[n] - c @ y[:n]) / l
        u = Li[:n, :n].T @ c
        inc = -np.outer(u / l, yn)
        x[:n] += inc
        x[n] = yn / l
        # two-sum of the increment into (hi, lo)
        a, b = xk[:n], inc
        s_ = a + b
        bb = s_ - a
        err = (a - (s_ - bb)) + (b - bb)
        xk[:n] = s_
        xk_lo[:n] += err
        xk[n] = yn / l
        xp[:n] += inc
        xp[n] = yn / l
        L[n, :n] = c
        L[n, n] = l
        Li[n, :n] = -u / l
        Li[n, n] = 1.0 / l
        y[n] = yn
        if (n + 1) % PERIOD == 0:
            xp[: n + 1] = Li[: n + 1, : n + 1].T @ y[: n + 1]
        if n % 500 == 0:
            print("append", n, flush=True)
    w_ref = F.solve(D)
    w_fresh = Li.T @ y
    w_refw = x + Li.T @ (y - L.T @ x)

    def rel(a, b):
        return float(np.abs(a - b).max() / np.abs(b).max())

    print("weights vs reference: inc %.3g fresh %.3g refw %.3g" % (rel(x, w_ref), rel(w_fresh, w_ref),
                                                                   rel(w_refw, w_ref)))
    print("factor L vs reference: %.3g" % rel(L, F.L))
    part = O.partition(wl.nb, 64, 0)
    group = part[29] if isinstance(part, list) else part[1][part[2][29]:part[2][30]]
    w_kahan = xk + xk_lo
    print("kahan %.3g periodic(%d) %.3g" % (rel(w_kahan, w_ref), PERIOD, rel(xp, w_ref)))
    for name, w in (("ref", w_ref), ("inc", x), ("fresh", w_fresh), ("refw", w_refw), ("kahan", w_kahan),
                    ("periodic", xp)):
        e = O.residual_errors(np.asarray(group), wl.points, wl.disp, P, w, R)
        top = np.argsort(-e)[:3]
        print(name, [(int(group[i]), float(e[i])) for i in top])


if __name__ == "__main__":
    main()
