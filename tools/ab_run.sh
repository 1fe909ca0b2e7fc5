#!/bin/bash
# Interleaved A/B of the ab/ library variants: tools/ab_run.sh ROUNDS NAME...
R=$1; shift
for r in $(seq $R); do
  for n in "$@"; do
    printf "%-8s " $n
    MEMPLAN_LIB=paper_1903_06631_b200/ab/lib_$n.so python tools/stage_probe.py --reps 10 2>&1 | grep -E "^  place  " | awk '{print $2}'
  done
done
