timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for t in CE SMPC1 SMPC3 SMPC8; do timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "loop.*"; done
for t in SMPC3 SMPC8; do TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree $t --iters 200 --reps 2 --skip-gap 2>&1 | tail -16; done
