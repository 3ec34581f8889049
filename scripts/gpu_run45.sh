export BFA_JIT_CACHE=/tmp/bfa_cold_$$
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 800 -k "work_queue" 2>&1 | tail -2
for QC in 4 16 64; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": 50, \"dual_pipe\": 1, \"queue_bodies\": 128, \"queue_classes\": $QC}"
echo "classes $QC"; timeout 1500 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1
done
