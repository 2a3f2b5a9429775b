"""Summarise `ncu --set full` reports: one row per captured kernel launch.

    python tools/ncu_summary.py report.ncu-rep [...] > profiles/xxx.md
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_inst_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "regs"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%"),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rdr = list(csv.reader(io.StringIO(out)))
    hdr, units = rdr[0], rdr[1]
    ix = {h: i for i, h in enumerate(hdr)}
    for r in rdr[2:]:
        rec = {"kernel": r[ix["Kernel Name"]][:60]}
        for m, name in METRICS:
            if m in ix:
                rec[name] = (r[ix[m]], units[ix[m]])
        yield rec


def main():
    print("| report | kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|" + "---|" * (len(METRICS) + 2))
    for p in sys.argv[1:]:
        for rec in rows(p):
            cells = [f"{rec.get(n, ('-', ''))[0]} {rec.get(n, ('-', ''))[1]}".strip() for _, n in METRICS]
            print(f"| {p.split('/')[-1]} | {rec['kernel']} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
