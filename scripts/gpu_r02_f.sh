#!/bin/bash
# round 2: GPU suite + bench line, then the ncu evidence (profiling pass of gpu_r02_d.sh)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_f.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
echo "bench rc=$?" >> gpurun_out/bench_f.err
bash scripts/gpu_r02_d.sh
