for B in '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "split_policy": 0}' \
         '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "split_policy": 1}' \
         '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "split_policy": 1, "streams": 8}' \
         '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "split_policy": 1, "streams": 16}'; do
echo "$B"
timeout 1500 python scripts/decomp.py c5 "$B" 4096,0 8192,0 2>&1 | tail -2
done
