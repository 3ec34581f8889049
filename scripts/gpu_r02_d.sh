#!/bin/bash
# round 2 profiling call: ncu evidence for the bench line (one GPU)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
M="gpu__time_duration.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,launch__registers_per_thread"
# (a) launch list of the bench command
B="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
$B > gpurun_out/d_bench_plain.json 2> gpurun_out/d_bench_plain.err &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/d_launches_bench.csv $B > gpurun_out/d_bench_ncu.log 2>&1
echo "a rc=$?" >> gpurun_out/d_status.txt
# (b) --set full of the headline kernel (C5 exhaustive) and of the C4 exhaustive kernel
for t in exhaustive c4_exhaustive; do
  python scripts/profile_target.py $t 2 > gpurun_out/d_plain_$t.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -s 1 -c 1 -o gpurun_out/d_full_$t python scripts/profile_target.py $t 2 > gpurun_out/d_ncu_$t.log 2>&1
  echo "b $t rc=$?" >> gpurun_out/d_status.txt
done
# (c) DRAM bytes of every materialised-mode kernel (one step per variant)
python scripts/profile_target.py materialised 1 > gpurun_out/d_plain_mat.log 2>&1 &&
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/d_mat_dram.csv python scripts/profile_target.py materialised 1 > gpurun_out/d_ncu_mat.log 2>&1
echo "c rc=$?" >> gpurun_out/d_status.txt
# (d) every work-queue module of the replay (direct call + replays)
python scripts/profile_target.py replay 3 > gpurun_out/d_plain_replay.log 2>&1 &&
ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/d_replay_modules.csv python scripts/profile_target.py replay 3 > gpurun_out/d_ncu_replay.log 2>&1
echo "d rc=$?" >> gpurun_out/d_status.txt
