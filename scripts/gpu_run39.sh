for QB in 256 1024; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"queue_bodies\": $QB}"
echo "queue_bodies $QB"; timeout 1200 python scripts/decomp.py c5 "$B" 16384,0 2>&1 | grep -v Traceback | tail -1
done
B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
echo "qb 512"; timeout 1200 python scripts/decomp.py c5 "$B" 16384,0 32768,0 2>&1 | grep -v Traceback | tail -2
