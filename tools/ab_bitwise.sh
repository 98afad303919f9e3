#!/bin/bash
# Bitwise HEAD (libtsmpc_head.so) vs working-tree build on the given trees, then timings.
# usage: tools/ab_bitwise.sh "W4k SMPC8 SMPC3" [iters]
trees=$1; it=${2:-60}
mkdir -p /tmp/ab
for t in $trees; do
  TSMPC_LIB=paper_1604_01074_b200/libtsmpc_head.so timeout 300 python tools/bitwise_variants.py --tree $t --iters $it --out /tmp/ab/h_$t.npz > /dev/null 2>&1
  echo "$t: $(timeout 300 python tools/bitwise_variants.py --tree $t --iters $it --out /tmp/ab/w_$t.npz --ref /tmp/ab/h_$t.npz 2>&1 | tail -1)"
done
