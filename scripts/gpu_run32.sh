B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1}'
timeout 2400 python scripts/decomp.py c5 "$B" 128,4 2048,0 1024,1 512,2 256,3 4096,0 1024,0 2>&1 | tail -8
