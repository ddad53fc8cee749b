#!/bin/bash
# round-end measurements (dev tool): bench lines of every workload + the C4 ncu captures
mkdir -p gpurun_out/fin2
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2/smoke.log 2>&1
for w in C4 C1 C2 C3 C5; do timeout 400 python bench.py --workload $w > gpurun_out/fin2/bench_$w.json 2> gpurun_out/fin2/bench_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin2/ncu_launches_c4.csv python bench.py --steps 2 --warmup 1 > gpurun_out/fin2/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k tsl_plan_kernel --csv --log-file gpurun_out/fin2/ncu_traffic_c4.csv python tools/ncu_one_build.py C4 > gpurun_out/fin2/ncu_tr4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k tsl_plan_kernel -c 1 -o gpurun_out/fin2/c4_full python tools/ncu_one_build.py C4 > gpurun_out/fin2/ncu_full.log 2>&1
python tools/stage_profile.py C4:70 C1 C2 > gpurun_out/fin2/stage.txt 2>&1
