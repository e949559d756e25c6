#!/bin/bash
# A/B timing of two in-tree builds (SGPX_LIB) in one GPU session: step timings, alternating.
#   tools/ab.sh libA.so libB.so [rounds]
cd "$(dirname "$0")/.."
for r in $(seq 1 ${3:-3}); do
  for lib in "$1" "$2"; do
    echo "$lib: $(SGPX_LIB=$lib python tools/profile_step.py --evals 10 2>&1 | tail -1)"
  done
done
