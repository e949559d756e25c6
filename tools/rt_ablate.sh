#!/bin/bash
# Row-tile kernel durations (forward, backward) under SGPX_RT_DBG timing experiments:
#   1 G = 0 stores only (no TMEM loads / exp2), 2 skip MMA3, 4 skip MMA1, 8 no exp2 math,
#   16 no operand streaming, 32 drain without TMEM loads.   usage: tools/rt_ablate.sh 0 1 2 ...
cd "$(dirname "$0")/.."
for d in "$@"; do
  t=$(SGPX_RT_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rowtile --csv \
      python tools/profile_step.py --evals 1 2>/dev/null | grep rowtile | awk -F, '{gsub(/"/,"",$NF); printf "%8.3f ", $NF/1e6}')
  echo "dbg=$d  fwd/bwd ms: $t"
done
