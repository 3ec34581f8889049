export BFA_JIT_CACHE=/tmp/bfa_cold_$$
B='{"slot_bits": 4, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 2400 python scripts/decomp.py c5 "$B" 16384,0 32768,0 2>&1 | grep -v Traceback | tail -2
B='{"slot_bits": 4, "inner_bits": 5, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 2400 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1
