"""Time the volume-kernel launch variants (RBF_EVAL_VARIANT) on configs[1]:
2M targets x 287 supports (or `--nv N --nc C`: the first N volume points,
C supports). One subprocess per variant (the variant is read once per
process)."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2004_04817_b200 as P
from paper_2004_04817_b200 import workloads as W
wl = W.config(1)
rng = np.random.default_rng(0)
NV, NC = int(sys.argv[1]), int(sys.argv[2])
idx = rng.choice(wl.nb, NC, replace=False)
sp = torch.from_numpy(wl.points[idx]).cuda(); sw = torch.from_numpy(rng.normal(size=(NC, 3)) * 0.01).cuda()
vol = torch.from_numpy(wl.volume[:NV]).cuda(); out = torch.empty_like(vol)
for _ in range(3): P.eval_device(vol, sp, sw, 2.0, deform=True, out=out)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.eval_device(vol, sp, sw, 2.0, deform=True, out=out); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(best)
'''
args = sys.argv[1:]
NV = int(args[args.index("--nv") + 1]) if "--nv" in args else 2_000_000
NC = int(args[args.index("--nc") + 1]) if "--nc" in args else 287
variants = [int(a) for a in args if a.isdigit() and (args.index(a) == 0 or args[args.index(a) - 1] not in ("--nv", "--nc"))]
res = {}
for v in variants or range(13):
    env = dict(os.environ, RBF_EVAL_VARIANT=str(v))
    r = subprocess.run([sys.executable, "-c", CODE, str(NV), str(NC)], env=env, capture_output=True, text=True)
    ms = float(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else None
    tf = 22 * NV * NC / (ms * 1e-3) / 1e12 if ms else None
    res[v] = {"ms": ms, "tflops": tf, "err": r.stderr[-300:] if r.returncode else ""}
    print(v, res[v], flush=True)
print(json.dumps(res))
