timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "graph or split_pieces or cofactoring or shard or autotune" 2>&1 | tail -3
for mb in 1 0; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"multi_body\": $mb}"
echo "multi_body $mb"; python scripts/decomp.py c5 "$B" 128,4 64,5 32,6 16,7 2>&1 | tail -4
done
