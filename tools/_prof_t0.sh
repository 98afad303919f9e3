TSMPC_TIMER_CTA=0 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap 2>&1 | tail -16 | grep -v " 0.00 us"
