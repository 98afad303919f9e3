#!/bin/bash
# Alternate HEAD (libtsmpc_head.so) and working-tree timings of the given trees.
for r in 1 2 3; do
  for t in "$@"; do
    a=$(TSMPC_LIB=paper_1604_01074_b200/libtsmpc_head.so timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    b=$(timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    echo "$t head $a | work $b"
  done
done
