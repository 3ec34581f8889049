#!/bin/bash
# ncu evidence for the end-of-round kernels (one GPU)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M="gpu__time_duration.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__registers_per_thread"
for t in exhaustive c4_exhaustive; do
  python scripts/profile_target.py $t 2 > gpurun_out/j_plain_$t.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -s 1 -c 1 -o gpurun_out/j_full_$t python scripts/profile_target.py $t 2 > gpurun_out/j_ncu_$t.log 2>&1
  echo "b $t rc=$?" >> gpurun_out/j_status.txt
done
python scripts/profile_target.py replay 3 > gpurun_out/j_plain_replay.log 2>&1 &&
ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/j_replay_modules.csv python scripts/profile_target.py replay 3 > gpurun_out/j_ncu_replay.log 2>&1
echo "d rc=$?" >> gpurun_out/j_status.txt
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$B > gpurun_out/j_bench_plain.json 2> gpurun_out/j_bench_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/j_launches_bench.csv $B > gpurun_out/j_bench_ncu.log 2>&1
echo "a rc=$?" >> gpurun_out/j_status.txt
