cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python scripts/autotune_objective.py 1 100 100000 > gpurun_out/autotune_objective.jsonl 2> gpurun_out/autotune_objective.err
echo "rc=$?" >> gpurun_out/autotune_objective.err
