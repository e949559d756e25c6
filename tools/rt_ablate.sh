#!/bin/bash
# Row-tile kernel durations (forward, backward) under SGPX_RT_DBG timing experiments:
#   1 skip the G math, 2 skip MMA3, 4 skip MMA1, 8 TMEM traffic without the exp2 math
#   (1/4/8 leave non-finite statistics, so only the kernels before the failing step are timed).
#   usage: tools/rt_ablate.sh 0 2 3 ...
cd "$(dirname "$0")/.."
for d in "$@"; do
  t=$(SGPX_RT_DBG=$d ncu --metrics gpu__time_duration.sum --clock-control none -k regex:rowtile --csv \
      python tools/profile_step.py --evals 1 2>/dev/null | grep rowtile | awk -F, '{gsub(/"/,"",$NF); printf "%8.3f ", $NF/1e6}')
  echo "dbg=$d  fwd/bwd ms: $t"
done
