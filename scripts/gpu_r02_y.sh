#!/bin/bash
# C4 count kernel at 2^12 .. 2^14 slot cofactors per thread-iteration
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/sweep_exhaustive.py c4 '[{"slot_bits": 12, "inner_bits": 0}, {"slot_bits": 13, "inner_bits": 0}, {"slot_bits": 13, "inner_bits": 0, "thread_bits": 7}, {"slot_bits": 14, "inner_bits": 0, "thread_bits": 7}, {"slot_bits": 14, "inner_bits": 0, "thread_bits": 6}, {"slot_bits": 12, "inner_bits": 0, "thread_bits": 7}, {"slot_bits": 13, "inner_bits": 1, "thread_bits": 7}]' > gpurun_out/y_c4_slots.jsonl 2> gpurun_out/y_c4_slots.err
echo "rc=$?" >> gpurun_out/y_c4_slots.err
