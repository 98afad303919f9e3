for r in 1 2; do
  for t in SMPC8; do
    a=$(TSMPC_LIB=paper_1604_01074_b200/libtsmpc_head.so timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    b=$(TSMPC_LIB=paper_1604_01074_b200/libtsmpc_cur.so timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    c=$(TSMPC_NO_AVG_OFFLOAD=1 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_cur.so timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "= .* us/iter")
    echo "$t head $a | offload $b | no-offload $c"
  done
done
