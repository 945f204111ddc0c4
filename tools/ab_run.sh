#!/bin/bash
# A/B timing of two library builds in one session (tools/ab/libA.so vs libB.so), alternating.
# Each variant is copied over the in-tree paper_1811_01277_b200/libelpa_b200.so for its run
# (the product binding loads only the in-tree build); the original is restored at the end.
# usage: tools/ab_run.sh OUT "SHAPES" cfg...
out=$1; shift; shapes=$1; shift
lib=paper_1811_01277_b200/libelpa_b200.so
cp $lib tools/ab/lib_orig.so
for round in 1 2; do
  for v in ${VARIANTS:-A B}; do
    cp tools/ab/lib$v.so $lib
    SHAPES="$shapes" REPS=${REPS:-5} timeout 600 python ${TOOL:-tools/quick_perf.py} "$@" | sed "s/^{/{\"lib\": \"$v\", \"round\": $round, /" >> $out
  done
done
cp tools/ab/lib_orig.so $lib
