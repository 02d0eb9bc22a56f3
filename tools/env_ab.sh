#!/bin/bash
# GPU A/B of environment knobs on the C5 bench: tools/env_ab.sh "SST_WF_POOL=4194304" "SST_WF_POOL=16777216 SST_WF_BATCH=2" ...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
k=0
for cfg in "$@"; do
  k=$((k+1))
  env $cfg timeout 300 python bench.py --no-cpu-baseline --no-extra ${AB_ARGS} > gpurun_out/env_$k.json 2> gpurun_out/env_$k.err
  python - "$cfg" "$k" <<'PY'
import json, sys
cfg, k = sys.argv[1], sys.argv[2]
try:
    d = json.loads(open(f"gpurun_out/env_{k}.json").read().strip().splitlines()[-1])
    e = d.get("e2e") or {}
    print(f"[{cfg}]", round(d["value"] / 1e9, 4), "e2e", round(e.get("value", 0) / 1e9, 4), round(d["ms_per_step"], 1),
          {k: round(x["ms"], 1) for k, x in d["roofline"]["kernels"].items()})
except Exception as ex:
    print(f"[{cfg}] FAILED", ex)
PY
done
