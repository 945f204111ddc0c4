#!/bin/bash
# Ablation timing of the two-group window kernel (development tool): each tools/ab/lib_abl<mask>.so
# (built with ELPA_B200_DEV_CFLAGS=-DKWIN_ABL=<mask>; wrong results, timing only) is copied over the
# in-tree library in turn; the original is restored at the end.
# usage: tools/abl_run.sh OUT "MASKS" cfg...
out=$1; shift; masks=$1; shift
lib=paper_1811_01277_b200/libelpa_b200.so
cp $lib tools/ab/lib_orig.so
for round in 1 2; do
  for m in $masks; do
    cp tools/ab/lib_abl$m.so $lib
    SHAPES="${SHAPES:-1,4,2,2}" REPS=${REPS:-3} timeout 600 python tools/quick_perf.py "$@" | grep shape | grep -v '"shape": null' | sed "s/^{/{\"abl\": $m, \"round\": $round, /" >> $out
  done
done
cp tools/ab/lib_orig.so $lib
