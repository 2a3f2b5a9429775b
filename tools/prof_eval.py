"""Volume kernel alone for ncu: configs[1]-sized (2M targets x 287 supports) or
configs[3]-sized (--nv, --nc), RBF_EVAL_VARIANT picks the launch variant.

    RBF_EVAL_VARIANT=0 ncu --set full -k regex:eval -c 1 python tools/prof_eval.py
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2004_04817_b200 as P  # noqa: E402
from paper_2004_04817_b200 import workloads as W  # noqa: E402

args = sys.argv[1:]
NV = int(args[args.index("--nv") + 1]) if "--nv" in args else 2_000_000
NC = int(args[args.index("--nc") + 1]) if "--nc" in args else 287
wl = W.config(1)
rng = np.random.default_rng(0)
idx = rng.choice(wl.nb, NC, replace=False)
sp = torch.from_numpy(wl.points[idx]).cuda()
sw = torch.from_numpy(rng.normal(size=(NC, 3)) * 0.01).cuda()
vol = torch.from_numpy(wl.volume[:NV]).cuda()
out = torch.empty_like(vol)
for _ in range(2):
    P.eval_device(vol, sp, sw, 2.0, deform=True, out=out)
torch.cuda.synchronize()
print("ok")
