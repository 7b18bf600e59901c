#!/bin/bash
# A/B of two library builds in one box session:
#   tools/ab_libs.sh <libA> <libB> "<B> <precision>" [rounds]
a=$1; b=$2; cfg=${3:-"512 1"}; rounds=${4:-2}
for r in $(seq $rounds); do
  for L in $a $b; do
    t=$(LSG_LIB=$L python tools/gen_forward.py ${cfg%% *} 20 ${cfg##* } | awk '{print $3}' | sort -n | head -1)
    echo "B/prec=$cfg lib=$L round=$r best=$t ms"
  done
done
