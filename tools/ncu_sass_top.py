"""Summarise an `ncu --page source --csv --print-source sass` dump: stall
reasons overall and the hottest SASS instructions by warp-stall samples."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ix = {h: i for i, h in enumerate(hdr)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = collections.Counter()
for r in data:
    for h in reasons:
        try:
            agg[h] += float(r[ix[h]] or 0)
        except ValueError:
            pass
print("total samples", tot)
for h, v in agg.most_common(12):
    print(f"  {h:28s} {v / tot * 100:6.1f}%")
top = sorted(data, key=lambda r: -float(r[ix[S]] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    best = max(reasons, key=lambda h: float(r[ix[h]] or 0))
    print(f"{r[ix['Address']]:>8} {float(r[ix[S]] or 0) / tot * 100:5.1f}% {best[6:]:14s} {r[ix['Source']][:90]}")
