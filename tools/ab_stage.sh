#!/bin/bash
# Interleaved A/B of ab/ variants on config-4 stage times: tools/ab_stage.sh ROUNDS "stage regex" NAME...
R=$1; shift; PAT=$1; shift
for r in $(seq $R); do
  for n in "$@"; do
    printf "%-8s " $n
    MEMPLAN_LIB=paper_1903_06631_b200/ab/lib_$n.so python tools/stage_probe.py --reps 10 2>&1 | grep -E "$PAT" | awk '{printf "%s %s  ", $1, $2} END {print ""}'
  done
done
