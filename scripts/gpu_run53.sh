B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 2400 python scripts/decomp.py c5 "$B" 32768,0 65536,0 2>&1 | grep -v Traceback | tail -2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); q=d['queue']; print(d['sp'], d['ms'], d['prep_s'], d['alu_floor_ms'], q['modules'], q['nvrtc_s'], q['bodies_s'])"
