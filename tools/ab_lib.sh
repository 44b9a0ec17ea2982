#!/usr/bin/env bash
# A/B of two library builds, alternating rounds (tools/qs_ab.py each):
#   bash tools/ab_lib.sh OUT libA.so libB.so "qs_ab args..."
OUT=gpurun_out/$1; A=$2; B=$3; ARGS=$4; mkdir -p $OUT
for r in 1 2; do
  for L in $A $B; do
    echo "== $L round $r" >> $OUT/ab.txt
    eval "PP_LIB_PATH=$PWD/$L timeout 400 python tools/qs_ab.py $ARGS --rounds 1" >> $OUT/ab.txt 2>&1
  done
done
