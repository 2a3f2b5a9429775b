"""Per-source-line warp-stall samples from `ncu --page source --csv
--print-source cuda,sass` (lines whose Address column is '-')."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
cur_file = None
out = []
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            s = float(r[4])
        except ValueError:
            continue
        if s > 0:
            out.append((s, cur_file, r[0], r[1]))
tot = sum(o[0] for o in out)
for s, f, ln, src in sorted(out, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{s / tot * 100:5.1f}% {f}:{ln:5s} {src.strip()[:100]}")
