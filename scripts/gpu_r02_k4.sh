#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python scripts/sweep_decomposed.py '[{"split_pieces": 4096, "queue_slot_bits": 7, "queue_inner": 1, "queue_role_budget": 50}, {"split_pieces": 6144, "queue_slot_bits": 7, "queue_inner": 1, "queue_role_budget": 50}, {"split_pieces": 8192, "queue_slot_bits": 6, "queue_inner": 1, "queue_role_budget": 50}, {"split_pieces": 4096, "queue_slot_bits": 6, "queue_inner": 2, "queue_role_budget": 75}, {"split_pieces": 6144, "queue_role_budget": 50}]' > gpurun_out/sweep_k4.jsonl 2> gpurun_out/sweep_k4.err
