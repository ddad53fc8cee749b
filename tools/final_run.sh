set -x
mkdir -p gpurun_out/fin
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/fin/gputests.log 2>&1; echo rc=$? >> gpurun_out/fin/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1
for w in C4 C1 C2 C3 C5; do timeout 400 python bench.py --workload $w > gpurun_out/fin/bench_$w.json 2> gpurun_out/fin/bench_$w.err; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin/ncu_launches_c4.csv python bench.py --steps 2 --warmup 1 > gpurun_out/fin/ncu_bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k tsl_plan_kernel --csv --log-file gpurun_out/fin/ncu_traffic_c4.csv python tools/ncu_one_build.py C4 > gpurun_out/fin/ncu_tr4.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k tsl_plan_kernel --csv --log-file gpurun_out/fin/ncu_traffic_c2.csv python tools/ncu_one_build.py C2 > gpurun_out/fin/ncu_tr2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k tsl_plan_kernel -c 1 -o gpurun_out/fin/c4_full python tools/ncu_one_build.py C4 > gpurun_out/fin/ncu_full.log 2>&1
ls -la gpurun_out/fin
