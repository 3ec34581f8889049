#!/bin/bash
# coalesced eval stores: the GPU suite, then the bench line (c4_eval extra)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/t_bench.json 2> gpurun_out/t_bench.err
echo "rc=$?" >> gpurun_out/t_bench.err
