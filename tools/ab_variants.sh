#!/bin/bash
# Time libtsmpc_<variant>.so builds against each other on one box, interleaved.
# usage: tools/ab_variants.sh "SMPC8 W4k" varA varB ...   (env per tree via TSMPC_* as usual)
trees=$1; shift
for r in 1 2; do
  for t in $trees; do
    for v in "$@"; do
      a=$(TSMPC_LIB=paper_1604_01074_b200/libtsmpc_$v.so timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
      echo "$t $v $a"
    done
  done
done
