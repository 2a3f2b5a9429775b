# Source-level ncu capture of the last configs[3] grid launch (n = 4096..4872), summarised
# on the box (per-line and per-SASS stall samples) so the report itself need not come back.
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gcb_grid -s 3 -c 1 -o gpurun_out/p3 python tools/sel_time.py --config 3 --reps 1 > gpurun_out/p3.log 2>&1
tail -2 gpurun_out/p3.log
ncu -i gpurun_out/p3.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/p3_src.csv 2>/dev/null
python tools/ncu_lines_top.py gpurun_out/p3_src.csv 45 > gpurun_out/p3_lines.txt
ncu -i gpurun_out/p3.ncu-rep --page source --csv --print-source sass > gpurun_out/p3_sass.csv 2>/dev/null
python tools/ncu_sass_top.py gpurun_out/p3_sass.csv 30 > gpurun_out/p3_sass.txt
python tools/ncu_summary.py gpurun_out/p3.ncu-rep > gpurun_out/p3_summary.md
rm -f gpurun_out/p3.ncu-rep gpurun_out/p3_src.csv gpurun_out/p3_sass.csv
cat gpurun_out/p3_summary.md; head -50 gpurun_out/p3_lines.txt
