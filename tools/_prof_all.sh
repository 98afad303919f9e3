timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for t in SMPC1 SMPC3; do timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "loop.*"; done
for t in SMPC1 SMPC3; do timeout 120 python tools/prof_case.py --tree $t --iters 500 --reps 3 --skip-gap 2>&1 | grep -o "loop.*"; done
TSMPC_TIMER_CTA=120 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap 2>&1 | tail -16 | grep -v " 0.00 us"
TSMPC_TIMER_CTA=120 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap 2>&1 | tail -16 | grep -v " 0.00 us"
