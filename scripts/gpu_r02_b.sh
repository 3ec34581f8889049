#!/bin/bash
# round 2: full GPU suite + bench + decomposed frontier sweep
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_full.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
echo "bench rc=$?" >> gpurun_out/bench_b.err
timeout 1500 python scripts/sweep_decomposed.py '[{"split_pieces": 4096}, {"split_pieces": 8192}, {"split_pieces": 16384}, {"split_pieces": 32768}, {"split_pieces": 16384, "slot_bits": 4}, {"split_pieces": 32768, "slot_bits": 4}]' > gpurun_out/sweep_b.jsonl 2> gpurun_out/sweep_b.err
echo "sweep rc=$?" >> gpurun_out/sweep_b.err
