# Round-2 evidence (final build) on one B200 (run from the repo root under gpurun): bench lines
# (ours + reference arm), ncu launch list of the bench command, full captures of
# the headline kernel (wide, SMPC8) and of the SMPC3 kernel, DRAM traffic, phase timers.
set -u
E=${E:-gpurun_out/ev5}
mkdir -p $E
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $E/smi.txt 2>&1
python tools/prof_case.py --tree SMPC8 --iters 50 --skip-gap > $E/plain8.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apg_wide_kernel -s 12 -c 1 -f \
  -o $E/wide_smpc8 python tools/prof_case.py --tree SMPC8 --iters 50 --skip-gap > $E/ncu_smpc8.log 2>&1
python tools/prof_case.py --tree SMPC3 --iters 50 --skip-gap > $E/plain3.log 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:apg_sparse_kernel -c 1 -f \
  -o $E/sparse_smpc3 python tools/prof_case.py --tree SMPC3 --iters 50 --skip-gap > $E/ncu_smpc3.log 2>&1
python tools/prof_case.py --tree W4k --iters 20 --skip-gap > $E/plainw4k.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:apg_wide_kernel -s 12 -c 1 -f \
  -o $E/wide_w4k python tools/prof_case.py --tree W4k --iters 20 --skip-gap > $E/ncu_w4k.log 2>&1
python tools/ncu_summary.py $E/wide_w4k.ncu-rep "python tools/prof_case.py --tree W4k --iters 20 --skip-gap" > $E/ncu_full_wide_w4k.txt 2>&1
python tools/ncu_traffic.py $E/wide_w4k.ncu-rep --tree W4k --iters 20 > $E/trafficw4k.log 2>&1
python tools/ncu_traffic.py $E/wide_smpc8.ncu-rep --tree SMPC8 --iters 50 > $E/traffic8.log 2>&1
python tools/ncu_traffic.py $E/sparse_smpc3.ncu-rep --tree SMPC3 --iters 50 > $E/traffic3.log 2>&1
cp profiles/ncu_traffic.json $E/ncu_traffic.json
python tools/ncu_summary.py $E/wide_smpc8.ncu-rep "python tools/prof_case.py --tree SMPC8 --iters 50 --skip-gap" > $E/ncu_full_wide_smpc8.txt 2>&1
python tools/ncu_summary.py $E/sparse_smpc3.ncu-rep "python tools/prof_case.py --tree SMPC3 --iters 50 --skip-gap" > $E/ncu_full_sparse_smpc3.txt 2>&1
# bench lines (after the traffic file is refreshed), as the driver runs them
timeout 900 python bench.py --steps 20 --warmup 5 > $E/bench.json 2> $E/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $E/bench_reference.json 2> $E/bench_reference.err
# launch list of the bench command (headline part)
python bench.py --steps 2 --warmup 1 --quick > $E/plain_bench.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file $E/launches.csv python bench.py --steps 2 --warmup 1 --quick > $E/ncu_launch.log 2>&1
python tools/ncu_launch_summary.py $E/launches.csv > $E/launches_summary.txt 2>&1
# phase timers (profiling build): a 4-chain chain CTA and a trunk CTA of SMPC8, a chain CTA of SMPC3
PROF_UNTUNED=1 TSMPC_TIMER_CTA=1 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC8 --iters 200 --reps 2 --skip-gap > $E/timers_smpc8_cta1.txt 2>&1
PROF_UNTUNED=1 TSMPC_TIMER_CTA=130 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC8 --iters 200 --reps 2 --skip-gap > $E/timers_smpc8_cta130.txt 2>&1
PROF_UNTUNED=1 TSMPC_TIMER_CTA=0 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap > $E/timers_smpc3_cta0.txt 2>&1
# the summaries above are what is kept; the reports stay on the box (gpurun_out/ is capped)
ls -la $E/*.ncu-rep > $E/reports.txt 2>&1
rm -f $E/*.ncu-rep
du -sh $E
tail -c 600 $E/bench.json; echo; tail -c 400 $E/bench_reference.json
