#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -k "exhaustive_bench or c1_posets or bench_multi_rank" > gpurun_out/pytest_n.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_n.log
timeout 1200 python bench.py > gpurun_out/bench_n.json 2> gpurun_out/bench_n.err
echo "bench rc=$?" >> gpurun_out/bench_n.err
