#!/bin/bash
# Round-end measurement set (run on the GPU box from the repo root):
# default bench line, the reference (CPU) arm, every BASELINE config, the
# configs[4] m-sweep, then the ncu evidence (launch list of the default bench
# command, full captures of the loop and volume kernels on configs[1] and of
# the grid loop kernel on configs[2]). Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py > gpurun_out/m_bench_cfg1.json 2> gpurun_out/m_bench_cfg1.err
  timeout 900 python bench.py --impl reference > gpurun_out/m_bench_ref.json 2> gpurun_out/m_bench_ref.err
  timeout 900 python bench.py --config 0 > gpurun_out/m_bench_cfg0.json 2> gpurun_out/m_bench_cfg0.err
  timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_cfg2.json 2> gpurun_out/m_bench_cfg2.err
  timeout 1500 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/m_bench_cfg3.json 2> gpurun_out/m_bench_cfg3.err
  timeout 900 python tools/msweep.py --out gpurun_out/m_msweep.json > gpurun_out/m_msweep.log 2>&1
  for f in gpurun_out/m_bench_*.json; do echo "$f: $(head -c 160 $f)"; done
fi
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/m_launches_cfg1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
      > gpurun_out/m_ncu_launches.log 2>&1
  # one selection = the one-cluster loop launch(es) + whole-GPU tail launches;
  # capture the first (longest) loop launch, the volume kernel, and the
  # configs[2] grid launches (the longest one is the loop)
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gcb_msg_kernel" \
      -s 0 -c 1 -o gpurun_out/m_prof_cfg1 python tools/prof_step.py --steps 1 > gpurun_out/m_ncu_cfg1.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"eval_kernel" \
      -s 0 -c 1 -o gpurun_out/m_prof_cfg1_eval python tools/prof_step.py --steps 1 > gpurun_out/m_ncu_cfg1_eval.log 2>&1
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"gcb_" \
      -s 0 -c 4 -o gpurun_out/m_prof_cfg2 python tools/prof_step.py --config 2 --steps 1 > gpurun_out/m_ncu_cfg2.log 2>&1
  if [ "${NCU_CFG3:-0}" = 1 ]; then
    timeout 1800 ncu --set full --clock-control none -k regex:"gcb_grid" \
        -s 0 -c 2 -o gpurun_out/m_prof_cfg3 python tools/prof_step.py --config 3 --steps 1 > gpurun_out/m_ncu_cfg3.log 2>&1
  fi
  tail -n 1 gpurun_out/m_ncu_cfg1.log gpurun_out/m_ncu_cfg1_eval.log gpurun_out/m_ncu_cfg2.log
fi
# keep what comes back small (gpurun merges at most 64 MiB): per-report raw CSV
# and the summary table on the box, then drop reports larger than 24 MiB
for r in gpurun_out/m_prof_*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}_raw.csv" 2>/dev/null
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}_details.csv" 2>/dev/null
done
python tools/ncu_summary.py gpurun_out/m_prof_*.ncu-rep > gpurun_out/m_ncu_summary.md 2>/dev/null
find gpurun_out -name 'm_prof_*.ncu-rep' -size +24M -delete
du -sh gpurun_out
