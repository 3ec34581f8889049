#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/profile_target.py exhaustive 2 > gpurun_out/o_plain_exhaustive.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -s 1 -c 1 -o gpurun_out/o_full_exhaustive python scripts/profile_target.py exhaustive 2 > gpurun_out/o_ncu_exhaustive.log 2>&1
echo "rc=$?" >> gpurun_out/o_ncu_exhaustive.log
