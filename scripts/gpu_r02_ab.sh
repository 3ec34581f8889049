#!/bin/bash
# launch list of the end-of-round bench command (first 600 launches), after
# the same command exits 0 without ncu
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 900 $B > gpurun_out/ab_bench.json 2> gpurun_out/ab_bench.err && echo "plain rc=0" >> gpurun_out/ab_bench.err &&
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/ab_launches_bench.csv $B > gpurun_out/ab_bench_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ab_bench_ncu.log
