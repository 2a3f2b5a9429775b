"""Displacement deviation of the volume-kernel pair forms from the reference
goldens (tests/golden/*.npz: the reference's own weights and displacements),
one process per RBF_EVAL_VARIANT (read once per process):

    RBF_EVAL_VARIANT=4 python tools/eval_form_accuracy.py   # difference form
    RBF_EVAL_VARIANT=7 python tools/eval_form_accuracy.py   # 64 x 6 launch shape
"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

G = Path(__file__).resolve().parent.parent / "tests" / "golden"
CASES = {"cfg0_m8": lambda: W.config(0, nv=100_000), "cfg1_m32": lambda: W.config(1, nv=2_000_000),
         "cfg2_m48": lambda: W.config(2, nv=200_000), "cfg3_m64_cap400": lambda: W.config(3, nv=100_000)}
for name, mk in CASES.items():
    g = np.load(G / f"{name}.npz")
    wl = mk()
    radius = float(g["params"][0])
    sup = P.SupportSet(g["seq"], wl.points[g["seq"]], g["weights"])
    u = P.evaluate_displacements(wl.volume[g["vol_idx"]], sup, radius)
    ref = g["vol_u"]
    rel = np.abs(u - ref).max() / np.abs(ref).max()
    wsum = np.abs(g["weights"]).sum(axis=0).max()
    print(f"{name:16s} variant {os.environ.get('RBF_EVAL_VARIANT', '4')}: max|du|/max|u| {rel:.2e}  "
          f"(sum|w| {wsum:.1e}, max|u| {np.abs(ref).max():.2e})")
