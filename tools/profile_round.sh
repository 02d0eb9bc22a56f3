#!/bin/bash
# One gpurun call that captures the round's profiling evidence for the CURRENT sources
# (each ncu run follows a plain run of the same command that exited 0):
#   gpurun_out/src_hash.txt          bench.source_hash() of the profiled build
#   gpurun_out/launches_bench.csv    ncu launch list (gpu__time_duration) of a short bench run
#   gpurun_out/launches_wf16.csv     ncu per-launch DRAM bytes of one 16-spp C5 render
#   gpurun_out/prof_wf.ncu-rep       ncu --set full of logic / trace / sphere / shadow (bulk iterations)
# then, here: tools/profile_summarize.sh <round> writes profiles/<round>/ and profiles/traffic.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import bench; print(bench.source_hash())" > gpurun_out/src_hash.txt
B="python bench.py --steps 2 --warmup 3 --no-frame --no-extra --no-e2e --no-cpu-baseline"
$B > gpurun_out/bench_short.json 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches_bench.csv \
      $B > gpurun_out/ncu_a.log 2>&1
echo "ncu launches rc=$?"
W="python tools/wf_prof.py st 16"
$W > gpurun_out/wfprof_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_wf16.csv $W > gpurun_out/ncu_b.log 2>&1
echo "ncu traffic rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_wf_(logic|trace|sphere|shadow)" -s 40 -c 5 \
    -o gpurun_out/prof_wf $W > gpurun_out/ncu_c.log 2>&1
echo "ncu full rc=$?"
# per-line stalls: ncu attributes the production build's inline-PTX evict_last loads to the
# asm lines, so the line view comes from a plain-__ldg build of the same sources
# (tools/build_variant.sh nokeep -DSST_L2_KEEP=0, built here from the current sources)
tools/build_variant.sh nokeep -DSST_L2_KEEP=0 > gpurun_out/build_nokeep.log 2>&1
if [ -f build_var/nokeep/libsst_gpu.so ]; then
  SST_GPU_LIB=build_var/nokeep/libsst_gpu.so ncu --set full --clock-control none --import-source on \
      -k regex:"k_wf_(logic|trace|sphere|shadow)" -s 40 -c 5 -o gpurun_out/prof_wf_lines $W > gpurun_out/ncu_d.log 2>&1
  echo "ncu lines rc=$?"
fi
