# W4k profiling on one B200 (run under gpurun from the repo root): plain run, phase timers of three CTAs,
# one ncu --set full capture of the wide kernel (untuned placement) and its summary.
set -u
E=gpurun_out/w4k
mkdir -p $E
timeout 300 python tools/prof_case.py --tree W4k --iters 100 --reps 2 --skip-gap > $E/plain.log 2>&1
for c in 0 60 147; do
TSMPC_TIMER_CTA=$c TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 300 python tools/prof_case.py --tree W4k --iters 100 --reps 2 --skip-gap > $E/timers_cta$c.txt 2>&1
done
PROF_UNTUNED=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:apg_wide_kernel -c 1 -f \
  -o $E/wide_w4k python tools/prof_case.py --tree W4k --iters 20 --skip-gap > $E/ncu.log 2>&1
python tools/ncu_summary.py $E/wide_w4k.ncu-rep "prof_case W4k 20 iters" > $E/ncu_full_wide_w4k.txt 2>&1
tail -3 $E/plain.log
