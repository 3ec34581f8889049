for Q in 1 4 16; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"queue_groups\": $Q}"
echo "queue_groups $Q"
timeout 1500 python scripts/decomp.py c5 "$B" 4096,0 2048,0 8192,0 2>&1 | tail -3
done
