"""Per-source-line stall breakdown (top reasons) from an ncu --set full report.
  python tools/ncu_line_stalls.py report.ncu-rep [top_lines] [file_filter]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
filt = sys.argv[3] if len(sys.argv) > 3 else ""
kf = sys.argv[4:] and ["-k", "regex:" + sys.argv[4]] or []
txt = subprocess.run(["ncu", "-i", rep] + kf + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot = defaultdict(float)
reasons = defaultdict(lambda: defaultdict(float))
src = {}
cur, hdr = "?", None
for row in csv.reader(io.StringIO(txt)):
    if not row:
        continue
    if row[0] == "File Path":
        cur = row[1].split("/")[-1]
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
    key = f"{cur}:{line}"
    src[key] = row[1].strip()[:70]
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h and h != "stall_selected":
            try:
                v = float(row[i] or 0)
            except ValueError:
                continue
            reasons[key][h[6:]] += v
            tot[key] += v
grand = sum(tot.values()) or 1
print(f"total stall samples {grand:.0f}")
for k in sorted(tot, key=tot.get, reverse=True)[:top]:
    if filt and filt not in k:
        continue
    r = sorted(reasons[k].items(), key=lambda x: -x[1])[:3]
    rs = " ".join(f"{n}={v / tot[k] * 100:.0f}%" for n, v in r)
    print(f"{k:22s} {tot[k] / grand * 100:5.1f}%  {rs:45s} {src[k]}")
