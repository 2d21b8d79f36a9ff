#!/bin/bash
# A/B of two library builds on one box: tools/ab_libs.sh A.so B.so cfg... (interleaved, 3 rounds)
A=$1; B=$2; shift 2
for r in 1 2 3; do
  for c in "$@"; do
    EB_LIB_PATH=$A python tools/prof_contract.py $c 10 lib=A | sed "s/\"variant\"/\"round\": $r, \"variant\"/"
    EB_LIB_PATH=$B python tools/prof_contract.py $c 10 lib=B | sed "s/\"variant\"/\"round\": $r, \"variant\"/"
  done
done
