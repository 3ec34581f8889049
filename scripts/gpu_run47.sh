B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 1500 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1 | cut -c1-300
B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512, "streams": 8}'
timeout 1500 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1 | cut -c1-300
