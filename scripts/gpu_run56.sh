timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1000 -k "work_queue or shard" 2>&1 | tail -2
B='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "queue_bodies": 512}'
timeout 2400 python scripts/decomp.py c5 "$B" 16384,0 32768,0 65536,0 2>&1 | grep -v Traceback | tail -3 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); q=d['queue']; print(d['sp'], d['ms'], d['count'], d['prep_s'], d['alu_floor_ms'], q['modules'], q['support_reduced'], q['chunks'])"
