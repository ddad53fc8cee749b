#!/bin/bash
# Round profile capture (run under gpurun): bench lines, the reference arm, the
# ncu launch list of the C2 bench, one full ncu capture of the planning kernel,
# the stage split, edge-case timings and executor replays.
set -u
mkdir -p gpurun_out/prof
for w in C1 C2 C3 C5; do
  timeout 300 python bench.py --workload $w > gpurun_out/prof/bench_${w,,}.json 2> gpurun_out/prof/bench_${w,,}.err
done
timeout 600 python bench.py --workload C4 --steps 1 --warmup 3 > gpurun_out/prof/bench_c4.json 2> gpurun_out/prof/bench_c4.err
timeout 300 python bench.py --impl reference > gpurun_out/prof/bench_reference_c2.json 2> gpurun_out/prof/bench_reference_c2.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof/ncu_launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
  > gpurun_out/prof/ncu_launch_run.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:tsl_plan_kernel -s 5 -c 1 \
  -o gpurun_out/prof/c2_full python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
  > gpurun_out/prof/ncu_full_run.log 2>&1
timeout 300 python tools/stage_profile.py C1 C2 C3 C5s0 edge:chain_x40 edge:C5.joint64 > gpurun_out/prof/stage_profile.txt 2>&1
timeout 300 python tools/edge_time.py > gpurun_out/prof/edge_time.txt 2>&1
timeout 300 python tools/exec_check.py C1 C2 C3 > gpurun_out/prof/executor_replay.txt 2>&1
ls -la gpurun_out/prof
