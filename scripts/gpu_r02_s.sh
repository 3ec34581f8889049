#!/bin/bash
# bench line with the C4 register-mode eval extra
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err
echo "rc=$?" >> gpurun_out/s_bench.err
