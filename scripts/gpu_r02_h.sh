#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_h.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_h.json 2> gpurun_out/bench_h.err
echo "bench rc=$?" >> gpurun_out/bench_h.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_h.json 2> gpurun_out/ref_h.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_h.log
