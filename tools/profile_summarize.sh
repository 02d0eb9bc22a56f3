#!/bin/bash
# Summaries of tools/profile_round.sh's captures into profiles/<round>/ (committed) and the
# src_hash-stamped profiles/traffic.json that bench.py reads.  tools/profile_summarize.sh r02
set -e
cd "$(dirname "$0")/.."
R=${1:-r02}
mkdir -p profiles/$R
H=$(cat gpurun_out/src_hash.txt)
python tools/launch_shares.py gpurun_out/launches_bench.csv profiles/$R/launch_shares_bench.json > /dev/null
gzip -c gpurun_out/launches_bench.csv > profiles/$R/launches_bench.csv.gz
gzip -c gpurun_out/launches_wf16.csv > profiles/$R/launches_wf16_traffic.csv.gz
python tools/traffic_summary.py gpurun_out/launches_wf16.csv profiles/traffic.json \
  "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none over every launch of one 16-spp C5 ST render (tools/wf_prof.py st 16), sources $H" "$H" > /dev/null
cp profiles/traffic.json profiles/$R/traffic.json
python tools/ncu_summary.py gpurun_out/prof_wf.ncu-rep --json profiles/$R/ncu_full_wavefront_summary.json > /dev/null
LREP=gpurun_out/prof_wf.ncu-rep
NOTE=""
if [ -f gpurun_out/prof_wf_lines.ncu-rep ]; then
  LREP=gpurun_out/prof_wf_lines.ncu-rep
  NOTE="# ncu --set full of a bulk launch on a build with plain __ldg gathers (SST_L2_KEEP=0): ncu attributes the inline-PTX evict_last loads of the production build to the asm lines, which hides the per-line picture; the kernels are otherwise identical."
fi
for k in logic trace sphere shadow; do
  { [ -n "$NOTE" ] && echo "$NOTE"; python tools/ncu_line_stalls.py $LREP 30 "" k_wf_$k; } > profiles/$R/ncu_full_k_wf_${k}_lines.txt
done
cp gpurun_out/wfprof_plain.log profiles/$R/wfprof_plain.log
echo "profiles/$R written for sources $H"
