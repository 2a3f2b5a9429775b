#!/bin/bash
# Round-end measurement set (run on the GPU box from the repo root):
# default bench line, the reference (CPU) arm, every BASELINE config, the
# configs[4] m-sweep. Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/m_bench_cfg1.json 2> gpurun_out/m_bench_cfg1.err
timeout 900 python bench.py --impl reference > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err
timeout 900 python bench.py --config 0 > gpurun_out/m_bench_cfg0.json 2> gpurun_out/m_bench_cfg0.err
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_cfg2.json 2> gpurun_out/m_bench_cfg2.err
timeout 1500 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_cfg3.json 2> gpurun_out/m_bench_cfg3.err
timeout 900 python tools/msweep.py --out gpurun_out/m_msweep.json > gpurun_out/m_msweep.log 2>&1
for f in gpurun_out/m_bench_*.json; do echo "$f: $(head -c 160 $f)"; done
