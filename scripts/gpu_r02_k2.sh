#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/c5_positions_2p28.py gpu profiles/r02/c5_positions_2p28.json > gpurun_out/k2_positions.log 2>&1
echo "rc=$?" >> gpurun_out/k2_positions.log
cp profiles/r02/c5_positions_2p28_gpu.json gpurun_out/ 2>/dev/null
