#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2700 python scripts/sweep_decomposed.py '[{"split_pieces": 4096, "queue_slot_bits": 7, "queue_role_budget": 50}, {"split_pieces": 4096, "queue_slot_bits": 7, "queue_role_budget": 30}, {"split_pieces": 3072, "queue_slot_bits": 7, "queue_role_budget": 50}, {"split_pieces": 8192, "queue_slot_bits": 7, "queue_role_budget": 50}, {"split_pieces": 16384, "queue_slot_bits": 7}]' > gpurun_out/sweep_q.jsonl 2> gpurun_out/sweep_q.err
echo "rc=$?" >> gpurun_out/sweep_q.err
