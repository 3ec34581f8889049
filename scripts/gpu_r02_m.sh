#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -k "decomposed or work_queue or concurrent or queue_options or count_shard or split_pieces" > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m.log
timeout 1500 python scripts/sweep_decomposed.py '[{}, {"split_pieces": 16384}, {"split_pieces": 8192}]' > gpurun_out/sweep_m.jsonl 2> gpurun_out/sweep_m.err
