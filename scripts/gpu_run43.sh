export BFA_JIT_CACHE=/tmp/bfa_cold_$$
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 800 -k "work_queue" 2>&1 | tail -3
B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 2400 python scripts/decomp.py c5 "$B" 16384,0 32768,0 2>&1 | grep -v Traceback | tail -2
