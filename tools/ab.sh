#!/bin/bash
# GPU A/B of library builds on the C5 bench (kernel-only line): tools/ab.sh main <variant> ...
# (main = the in-tree library; others = build_var/<name>/libsst_gpu.so from tools/build_variant.sh)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = main ]; then unset SST_GPU_LIB; else export SST_GPU_LIB=build_var/$v/libsst_gpu.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-extra ${AB_ARGS} > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/ab_{v}.json").read().strip().splitlines()[-1])
    print(v, round(d["value"] / 1e9, 4), {k: round(x["ms"], 1) for k, x in d["roofline"]["kernels"].items()})
except Exception as e:
    print(v, "FAILED", e)
PY
done
