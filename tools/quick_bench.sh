#!/bin/bash
# One compact line per bench run (GPU box): ms/step, e2e ms/step, selection
# ms, volume ms and the loop's per-phase microseconds. Usage: bash
# tools/quick_bench.sh [runs] [bench args...]
mkdir -p gpurun_out
runs=${1:-1}; shift
for i in $(seq 1 "$runs"); do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline "$@" > gpurun_out/qb$i.json 2>gpurun_out/qb$i.err
  python - "$i" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/qb{sys.argv[1]}.json").read().strip().splitlines()[-1])
b = d["breakdown"]
print(round(d["ms_per_step"], 4), round(d["e2e"]["ms_per_step"], 4), round(b["selection_ms"], 4),
      round(b["volume_ms"], 4), {k: round(v, 1) for k, v in b["loop_phase_us"].items()})
PY
done
