"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum)
from ncu reports, written to profiles/ncu_traffic.json for bench.py's
roofline "traffic" field.

    python tools/ncu_traffic.py report.ncu-rep [...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    out = {}
    for path in sys.argv[1:]:
        raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        ix = {h: i for i, h in enumerate(hdr)}
        for r in rows[2:]:
            name = r[ix["Kernel Name"]]
            key = "gcb_kernel" if "gcb_" in name else ("eval_kernel" if "eval_kernel" in name else name[:40])
            total = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                total += float(r[ix[m]]) * UNIT.get(units[ix[m]], 1)
            out[key] = {"bytes_per_launch": total, "report": Path(path).name, "kernel": name[:80]}
    dst = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
    dst.write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
