#!/bin/bash
# On the GPU box after round_measure.sh's ncu captures: summarise every
# report into text (per-launch metric table, DRAM traffic, full details CSV)
# and drop the largest .ncu-rep files until gpurun_out/ fits gpurun's 64 MiB
# copy-back limit.
set -u
out=gpurun_out/m_ncu_summary.md
: > "$out"
for r in gpurun_out/m_prof_*.ncu-rep; do
  python tools/ncu_summary.py "$r" >> "$out" 2>&1
  ncu -i "$r" --page details --csv > "${r%.ncu-rep}_details.csv" 2>/dev/null
done
python tools/ncu_traffic.py gpurun_out/m_prof_cfg1.ncu-rep gpurun_out/m_prof_cfg1_eval.ncu-rep > gpurun_out/m_ncu_traffic.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/m_ncu_traffic.json
while [ "$(du -sm gpurun_out | cut -f1)" -gt 56 ]; do
  big=$(ls -S gpurun_out/*.ncu-rep 2>/dev/null | head -1)
  [ -z "$big" ] && break
  rm -f "$big"
done
du -sh gpurun_out
