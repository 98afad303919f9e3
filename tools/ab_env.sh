#!/bin/bash
# Same library, environment switches A/B (read at plan creation), interleaved on one box.
# usage: tools/ab_env.sh "SMPC8 SMPC3" "TSMPC_NO_TOPS=1" ""   ("" = defaults)
trees=$1; shift
for r in 1 2; do
  for t in $trees; do
    for v in "$@"; do
      a=$(env $v timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
      echo "$t [$v] $a"
    done
  done
done
