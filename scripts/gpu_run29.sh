for st in 4 8 16; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"streams\": $st}"
echo "streams $st"; python scripts/decomp.py c5 "$B" 128,4 64,4 2>&1 | tail -2
done
