"""Where and why the configs[3] support sequence leaves the reference's.

Runs the device selection on configs[3] (Nb = 200k, R = 4, m = 64) capped just
before the first position where it differs from the reference golden
(tests/golden/cfg3_m64.npz), then scans the group the next iteration visits with
the device's weights at that point: prints the group's top candidates, the
error of the node the reference picked and the gap to ours, against the error
evaluation's own uncertainty (displacement spread of two stable solves, recorded
in the golden). Writes gpurun_out/cfg3_divergence.json.

    python tools/cfg3_divergence.py
"""

import json
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))


def main():
    import paper_2004_04817_b200 as P
    from paper_2004_04817_b200 import workloads as W
    from paper_2004_04817_b200.selection import _errors_at

    g = dict(np.load(REPO / "tests/golden/cfg3_m64.npz"))
    wl = W.config(3, nv=10)
    b = P.BoundarySet(np.arange(wl.nb), wl.points, wl.disp)
    full = P.gcb_select(b, P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=wl.nb, m=64))
    seq = np.asarray(full.support.nodes)
    k = min(len(seq), len(g["seq"]))
    d = np.flatnonzero(seq[:k] != g["seq"][:k])
    if not len(d):
        print("sequences identical")
        return
    first = int(d[0])
    capped = P.gcb_select(b, P.SelectionConfig(radius=wl.radius, tol=wl.tol, max_supports=first, m=64))
    assert np.array_equal(np.asarray(capped.support.nodes), g["seq"][:first])
    # the record that added support number `first` in the reference
    added = np.flatnonzero(np.isin(g["rec_node"], g["seq"][first:first + 1]))
    rec = int(added[0])
    group = int(g["rec_group"][rec])
    part = P.partition_boundary(b, 64, 0)
    members = np.asarray(part.groups[group])
    errs = _errors_at(members, b, capped.support.points, capped.support.weights, wl.radius)
    order = np.argsort(-errs)[:8]
    ref_node, our_node = int(g["seq"][first]), int(seq[first])
    e_ref = float(errs[np.flatnonzero(members == ref_node)[0]])
    e_our = float(errs[np.flatnonzero(members == our_node)[0]])
    noise = float(g["alt_u_rel"]) * float(np.abs(g["vol_u"]).max())
    out = {"first_difference": first, "record": rec, "group": group, "ref_node": ref_node,
           "our_node": our_node, "err_ref_node": e_ref, "err_our_node": e_our,
           "gap_rel": abs(e_our - e_ref) / max(e_our, e_ref),
           "displacement_noise_abs": noise, "ref_local_max": float(g["rec_local_max"][rec]),
           "top": [(int(members[i]), float(errs[i])) for i in order]}
    print(json.dumps(out, indent=1))
    (REPO / "gpurun_out").mkdir(exist_ok=True)
    (REPO / "gpurun_out" / "cfg3_divergence.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
