#!/bin/bash
# C4 count kernel at 2^9 / 2^10 slot cofactors per thread-iteration
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sweep_exhaustive.py c4 '[{}, {"slot_bits": 9, "inner_bits": 1}, {"slot_bits": 9, "inner_bits": 2}, {"slot_bits": 10, "inner_bits": 1}, {"slot_bits": 10, "inner_bits": 2}, {"slot_bits": 9, "inner_bits": 1, "thread_bits": 7}, {"slot_bits": 10, "inner_bits": 0}, {}]' > gpurun_out/w_c4_slots.jsonl 2> gpurun_out/w_c4_slots.err
echo "rc=$?" >> gpurun_out/w_c4_slots.err
