mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 1200 -k "not full_set_bits" 2>&1 | tail -4
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
python -c "
import json; d=json.load(open('gpurun_out/bench3.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'])
for c in d['autotune']['candidates']: print(c)
"
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench3_c4.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench3_c4.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['autotune']['best'])
for c in d['autotune']['candidates']: print(c)
"
