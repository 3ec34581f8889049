B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1}'
python scripts/decomp.py c5 "$B" 16,5 32,4 32,5 16,6 64,3 64,4 8,7 128,2 2>&1 | tail -9
