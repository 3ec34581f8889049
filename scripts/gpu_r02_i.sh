#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_i.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_i.json 2> gpurun_out/bench_i.err
echo "bench rc=$?" >> gpurun_out/bench_i.err
python scripts/sweep_exhaustive.py c5 '[{}, {"role_seeds": 1}, {"slot_bits": 6, "inner_bits": 3}]' > gpurun_out/sweep_exh_i.jsonl 2>&1
