"""Per-source-line aggregation of an ncu source page (cuda,sass correlation):
instructions executed, thread-instructions, stall samples.
  python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(lambda: [0, 0, 0, ""])
cur_file = "?"
hdr = None
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Function Name":
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    try:
        line = int(row[0])
    except ValueError:
        continue
    def g(name):
        try:
            return float(row[hdr.index(name)] or 0)
        except (ValueError, IndexError):
            return 0.0
    key = (cur_file, line)
    a = agg[key]
    a[0] += g("Instructions Executed")
    a[1] += g("Thread Instructions Executed")
    a[2] += g("Warp Stall Sampling (All Samples)")
    a[3] = row[1][:70]
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[2] for v in agg.values()) or 1
print(f"total warp-inst {tot_i:.3g}, stall samples {tot_s:.3g}")
print(f"{'file:line':28s} {'inst%':>6s} {'thr/inst':>8s} {'samp%':>6s}  source")
for (f, l), (i, t, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][2])[:top]:
    print(f"{f + ':' + str(l):28s} {100 * i / tot_i:6.2f} {t / max(i, 1):8.2f} {100 * s / tot_s:6.2f}  {src}")
