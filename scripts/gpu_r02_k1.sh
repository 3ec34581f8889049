#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python scripts/sweep_decomposed.py '[{}, {"queue_opt_level": 1}, {"queue_role_budget": 50}, {"split_pieces": 16384}, {"split_pieces": 16384, "queue_opt_level": 1, "queue_role_budget": 50}]' > gpurun_out/sweep_k.jsonl 2> gpurun_out/sweep_k.err
