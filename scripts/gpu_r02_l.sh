#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/sweep_exhaustive.py c5 '[{"role_budget": 800}, {"role_seeds": 6}, {"imad_cost_pct": 40}, {"imad_cost_pct": 60}, {"thread_bits": 7}, {"role_budget": 800, "role_seeds": 6}]' > gpurun_out/sweep_exh_l.jsonl 2>&1
python scripts/sweep_exhaustive.py c4 '[{}, {"role_seeds": 3}, {"slot_bits": 8, "inner_bits": 3}, {"thread_bits": 7}]' >> gpurun_out/sweep_exh_l.jsonl 2>&1
