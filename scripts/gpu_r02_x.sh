#!/bin/bash
# C4 count kernel at 2^11 / 2^12 slot cofactors per thread-iteration
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sweep_exhaustive.py c4 '[{"slot_bits": 10, "inner_bits": 1}, {"slot_bits": 11, "inner_bits": 1}, {"slot_bits": 11, "inner_bits": 0}, {"slot_bits": 12, "inner_bits": 1}, {"slot_bits": 12, "inner_bits": 0}, {"slot_bits": 11, "inner_bits": 1, "thread_bits": 7}, {"slot_bits": 12, "inner_bits": 1, "thread_bits": 7}, {"slot_bits": 10, "inner_bits": 1, "role_budget": 400}, {"slot_bits": 11, "inner_bits": 1, "role_budget": 400}]' > gpurun_out/x_c4_slots.jsonl 2> gpurun_out/x_c4_slots.err
echo "rc=$?" >> gpurun_out/x_c4_slots.err
