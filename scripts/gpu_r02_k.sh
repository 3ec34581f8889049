#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/c5_positions_2p28.py gpu profiles/r02/c5_positions_2p28.json > gpurun_out/k_positions.log 2>&1
cp profiles/r02/c5_positions_2p28_gpu.json gpurun_out/ 2>/dev/null
timeout 2400 python scripts/sweep_decomposed.py '[{}, {"queue_opt_level": 1}, {"queue_role_budget": 50}, {"split_pieces": 16384}, {"split_pieces": 16384, "queue_opt_level": 1, "queue_role_budget": 50}]' > gpurun_out/sweep_k.jsonl 2> gpurun_out/sweep_k.err
