B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1}'
timeout 1500 python scripts/decomp.py c5 "$B" 128,4 4096,0 2048,0 1024,0 2>&1 | tail -4
