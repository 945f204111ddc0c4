#!/bin/bash
# A/B timing of two library builds in one session (tools/ab/libA.so vs libB.so), alternating.
# usage: tools/ab_run.sh OUT "SHAPES" cfg...
out=$1; shift; shapes=$1; shift
for round in 1 2; do
  for v in A B; do
    ELPA_B200_LIB=tools/ab/lib$v.so SHAPES="$shapes" REPS=${REPS:-5} timeout 600 python ${TOOL:-tools/quick_perf.py} "$@" | sed "s/^{/{\"lib\": \"$v\", \"round\": $round, /" >> $out
  done
done
