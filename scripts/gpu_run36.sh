# cold JIT cache: measure preparation honestly
export BFA_JIT_CACHE=/tmp/bfa_cold_$$
for QB in 128 512; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"queue_bodies\": $QB}"
echo "queue_bodies $QB"
timeout 1200 python scripts/decomp.py c5 "$B" 8192,0 16384,0 2>&1 | grep -v Traceback | tail -4
done
