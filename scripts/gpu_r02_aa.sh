#!/bin/bash
# ncu of the slot-14 C4 kernel, then a bench line (eval against the measured store bandwidth)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/profile_target.py c4_exhaustive 2 > gpurun_out/aa_plain_c4.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -s 1 -c 1 -o gpurun_out/aa_full_c4 python scripts/profile_target.py c4_exhaustive 2 > gpurun_out/aa_ncu_c4.log 2>&1
echo "rc=$?" >> gpurun_out/aa_ncu_c4.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/aa_bench.json 2> gpurun_out/aa_bench.err
echo "rc=$?" >> gpurun_out/aa_bench.err
