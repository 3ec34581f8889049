#!/bin/bash
# kind-2 IMAD cells (option imad_pairs) against the preset, full-cube counts
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/sweep_exhaustive.py c5 '[{}, {"imad_pairs": 1}, {"imad_pairs": 1, "role_seed": 3}, {"imad_pairs": 1, "role_seed": 6}, {"imad_pairs": 2}, {"imad_pairs": 2, "role_seeds": 1}, {"imad_pairs": 1, "role_seeds": 1, "role_seed": 1}, {"imad_pairs": 1, "role_seeds": 1, "role_seed": 13}, {"imad_pairs": 1, "role_budget": 1600}]' > gpurun_out/v_pairs_c5.jsonl 2> gpurun_out/v_pairs_c5.err
echo "rc=$?" >> gpurun_out/v_pairs_c5.err
timeout 300 python scripts/sweep_exhaustive.py c4 '[{}, {"imad_pairs": 1}, {"imad_pairs": 2}]' > gpurun_out/v_pairs_c4.jsonl 2> gpurun_out/v_pairs_c4.err
echo "rc=$?" >> gpurun_out/v_pairs_c4.err
