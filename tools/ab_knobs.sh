#!/bin/bash
# A/B of generator launch knobs (LSG_GEN_KNOBS) in one box session:
#   tools/ab_knobs.sh "<B> <precision>" "<knob values>" [rounds]
# prints the best-of-20 forward time per knob value, rounds interleaved.
cfg=${1:-"128 0"}; knobs=${2:-"0 1 2 3"}; rounds=${3:-2}
for r in $(seq $rounds); do
  for k in $knobs; do
    t=$(LSG_GEN_KNOBS=$k python tools/gen_forward.py ${cfg%% *} 20 ${cfg##* } | awk '{print $3}' | sort -n | head -1)
    echo "B/prec=$cfg knobs=$k round=$r best=$t ms"
  done
done
