#!/bin/bash
# One gpurun call for the round's evidence at the current sources: profile_round.sh's ncu
# captures, the src_hash-stamped traffic file (so the bench line below reports it), the GPU
# test suite, smoke, the default bench line and the reference arm. Summarise afterwards
# with tools/profile_summarize.sh <round>.
cd "$(dirname "$0")/.."
tools/profile_round.sh
H=$(cat gpurun_out/src_hash.txt)
python tools/traffic_summary.py gpurun_out/launches_wf16.csv profiles/traffic.json \
  "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none over every launch of one 16-spp C5 ST render (tools/wf_prof.py st 16), sources $H" "$H" > /dev/null
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "gpu tests rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
