#!/bin/bash
# Split-mode trunk CTA count sweep (TSMPC_TRUNK_CTAS, read at plan creation), same box.
for r in 1 2; do
  for n in 20 26 34 40; do
    a=$(TSMPC_TRUNK_CTAS=$n timeout 120 python tools/prof_case.py --tree SMPC3 --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    echo "SMPC3 trunk_ctas=$n $a"
  done
  for n in 16 24 32; do
    a=$(TSMPC_TRUNK_CTAS=$n timeout 120 python tools/prof_case.py --tree SMPC8 --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    echo "SMPC8 trunk_ctas=$n $a"
  done
done
