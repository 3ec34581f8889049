for B in '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512, "role_budget": 400}' \
         '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512, "split_policy": 0}'; do
echo "$B"; timeout 1500 python scripts/decomp.py c5 "$B" 32768,0 2>&1 | grep -v Traceback | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); q=d['queue']; print(d['ms'], d['count'], d['prep_s'], d['alu_floor_ms'], q['bodies_s'], q['nvrtc_s'])"
done
