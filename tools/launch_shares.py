"""Kernel shares of an ncu launch list (--metrics gpu__time_duration.sum --csv):
  python tools/launch_shares.py launches.csv [out.json]
ncu times are cold-cache and serialised: compare SHARES with bench.py's per-kernel pass."""
import collections
import csv
import json
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if r[h.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"[<(].*", "", r[h.index("Kernel Name")]).replace("void ", "").strip()
    v = float(r[h.index("Metric Value")].replace(",", ""))
    unit = r[h.index("Metric Unit")]
    ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
    agg[name][0] += 1
    agg[name][1] += ns
tot = sum(v[1] for v in agg.values())
out = {k: {"launches": n, "ms": ns / 1e6, "share": ns / tot} for k, (n, ns) in
       sorted(agg.items(), key=lambda kv: -kv[1][1])}
print(json.dumps(out, indent=1))
if len(sys.argv) > 2:
    json.dump({"source": sys.argv[1], "kernels": out}, open(sys.argv[2], "w"), indent=1)
