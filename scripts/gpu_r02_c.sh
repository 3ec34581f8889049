#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
echo "bench rc=$?" >> gpurun_out/bench_c.err
timeout 600 python bench.py --steps 10 --warmup 3 --no-extras --no-cpu-baseline --options '{"role_budget": 400}' > gpurun_out/bench_c_rb400.json 2>> gpurun_out/bench_c.err
timeout 1500 python scripts/sweep_decomposed.py '[{"split_pieces": 32768, "queue_bodies": 256}, {"split_pieces": 16384, "queue_bodies": 256}, {"split_pieces": 32768, "queue_bodies": 256, "queue_light_pct": 30}, {"split_pieces": 8192, "queue_bodies": 256}]' > gpurun_out/sweep_c.jsonl 2> gpurun_out/sweep_c.err
echo "sweep rc=$?" >> gpurun_out/sweep_c.err
