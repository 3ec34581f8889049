mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout 1500 -k "not full_set_bits" 2>&1 | tail -4
python scripts/tune.py c5 38 "dual_pipe=0,role_search=0" "slot_bits=5,imad_cost_pct=35,role_search=0" "slot_bits=5,imad_cost_pct=35" "slot_bits=3,imad_cost_pct=50" "slot_bits=4,imad_cost_pct=35" "slot_bits=5,imad_cost_pct=50" "slot_bits=3,dual_pipe=0" 2>&1 | cut -c1-250
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench9.json 2> gpurun_out/bench9.err; tail -3 gpurun_out/bench9.err
python -c "
import json; d=json.load(open('gpurun_out/bench9.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'])
"
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench9_c4.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench9_c4.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'])
"
