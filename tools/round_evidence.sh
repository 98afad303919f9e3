# Round evidence on one B200 (run from the repo root under gpurun):
#   bench (ours + reference arm), ncu launch list, ncu full captures, DRAM traffic.
set -u
mkdir -p gpurun_out/ev
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/ev/smi.txt 2>&1
# DRAM traffic + full capture of the headline kernel (50 iterations, SMPC3), then SMPC8 and the gap kernels
timeout 600 ncu --set full --import-source on --clock-control none -k apg_sparse_kernel -c 1 -f \
  -o gpurun_out/ev/sparse_smpc3 python tools/prof_case.py --tree SMPC3 --iters 50 --skip-gap > gpurun_out/ev/ncu_smpc3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k apg_sparse_kernel -c 1 -f \
  -o gpurun_out/ev/sparse_smpc8 python tools/prof_case.py --tree SMPC8 --iters 50 --skip-gap > gpurun_out/ev/ncu_smpc8.log 2>&1
python tools/ncu_traffic.py gpurun_out/ev/sparse_smpc3.ncu-rep --tree SMPC3 --iters 50 > gpurun_out/ev/traffic3.log 2>&1
python tools/ncu_traffic.py gpurun_out/ev/sparse_smpc8.ncu-rep --tree SMPC8 --iters 50 > gpurun_out/ev/traffic8.log 2>&1
cp profiles/ncu_traffic.json gpurun_out/ev/ncu_traffic.json
python tools/ncu_summary.py gpurun_out/ev/sparse_smpc3.ncu-rep "python tools/prof_case.py --tree SMPC3 --iters 50 --skip-gap" > gpurun_out/ev/ncu_full_sparse_smpc3.txt 2>&1
python tools/ncu_summary.py gpurun_out/ev/sparse_smpc8.ncu-rep "python tools/prof_case.py --tree SMPC8 --iters 50 --skip-gap" > gpurun_out/ev/ncu_full_sparse_smpc8.txt 2>&1
# bench lines (after the traffic file is refreshed)
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err
# launch list of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/ev/launches.csv python bench.py --steps 2 --warmup 1 --no-sweep --no-cpu --no-shard --no-closed-loop > gpurun_out/ev/ncu_launch.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/ev/launches.csv > gpurun_out/ev/launches_summary.txt 2>&1
# phase timers (profiling build) of a chain CTA and a trunk CTA
TSMPC_TIMER_CTA=0 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap > gpurun_out/ev/timers_smpc3_cta0.txt 2>&1
TSMPC_TIMER_CTA=120 TSMPC_LIB=paper_1604_01074_b200/libtsmpc_timers.so timeout 120 python tools/prof_case.py --tree SMPC3 --iters 200 --reps 2 --skip-gap > gpurun_out/ev/timers_smpc3_cta120.txt 2>&1
tail -c 400 gpurun_out/ev/bench.json; echo; tail -c 300 gpurun_out/ev/bench_reference.json
