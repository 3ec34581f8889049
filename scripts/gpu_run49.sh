for IC in 35 65; do
B="{\"slot_bits\": 5, \"inner_bits\": 4, \"imad_cost_pct\": $IC, \"dual_pipe\": 1, \"queue_bodies\": 512}"
echo "imad $IC"; timeout 1500 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); q=d['queue']; print(d['ms'], d['prep_s'], d['alu_floor_ms'], d['cells_lop3'], d['cells_imad'])"
done
