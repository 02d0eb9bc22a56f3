"""Per-source-line breakdown of one stall reason from an ncu source page.
  python tools/ncu_stall_lines.py report.ncu-rep stall_no_inst [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, col = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(float)
src = {}
cur = "?"
hdr = None
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr) or row[0] == "Function Name":
        continue
    try:
        line = int(row[0])
        v = float(row[hdr.index(col)] or 0)
    except (ValueError, IndexError):
        continue
    agg[(cur, line)] += v
    src[(cur, line)] = row[1][:70]
tot = sum(agg.values()) or 1
by_file = defaultdict(float)
for (f, l), v in agg.items():
    by_file[f] += v
print("by file:", {f: round(100 * v / tot, 1) for f, v in sorted(by_file.items(), key=lambda x: -x[1])})
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{k[0] + ':' + str(k[1]):28s} {100 * v / tot:6.2f}%  {src[k]}")
