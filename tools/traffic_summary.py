"""Per-kernel-kind average DRAM traffic per launch from an ncu CSV launch list
(--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum):
  python tools/traffic_summary.py launches.csv out.json [source-note] [src_hash]
src_hash (bench.source_hash() of the sources the captured library was built from) is
stamped into the output; bench.py reports `roofline.traffic` only from a file whose
stamp matches the sources it runs.
"""
import collections
import csv
import json
import sys

KINDS = {"k_wf_logic": "wf_logic", "k_wf_gen": "wf_gen", "k_wf_trace": "wf_trace", "k_wf_sphere": "wf_sphere",
         "k_wf_shadow": "wf_shadow", "k_wf_reset": "wf_reset", "k_trace": "megakernel", "k_film": "film",
         "k_wf_compact": "wf_tail", "k_wf_init": "wf_init"}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
per = collections.defaultdict(dict)
for r in rows[hi + 1:]:
    per[(int(r[h.index("ID")]), r[h.index("Kernel Name")])][r[h.index("Metric Name")]] = float(
        r[h.index("Metric Value")].replace(",", ""))
agg = collections.defaultdict(lambda: collections.Counter())
for (i, name), m in per.items():
    kind = next((v for k, v in KINDS.items() if k in name), None)
    if kind is None:
        continue
    a = agg[kind]
    a["launches"] += 1
    a["bytes"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    a["ns"] += m.get("gpu__time_duration.sum", 0)
out = {"source": sys.argv[3] if len(sys.argv) > 3 else sys.argv[1], "kernels": {}}
if len(sys.argv) > 4:
    out["src_hash"] = sys.argv[4]
for k, a in agg.items():
    out["kernels"][k] = {"launches": a["launches"], "dram_bytes_per_launch": a["bytes"] / a["launches"],
                         "ncu_avg_us": a["ns"] / a["launches"] / 1e3}
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
