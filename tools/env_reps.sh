#!/bin/bash
# GPU A/B of environment knobs by repeated timed regions in one process (tools/timed_reps.py:
# K asynchronous C5 slabs x R repetitions): tools/env_reps.sh "SST_WF_TAIL=262144" "SST_WF_TAIL=1048576" ...
cd "$(dirname "$0")/.."
for cfg in "$@"; do
  echo "[$cfg] $(env $cfg timeout 300 python tools/timed_reps.py ${REPS:-3} ${STEPS:-10} 2>/dev/null | tail -1)"
done
