for C in 131072 524288 2097152; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"queue_bodies\": 512, \"queue_chunk\": $C}"
echo "queue_chunk $C"
timeout 1200 python scripts/decomp.py c5 "$B" 16384,0 2>&1 | grep -v Traceback | tail -1
done
