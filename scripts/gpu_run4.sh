mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; tail -3 gpurun_out/bench4.err
python -c "
import json; d=json.load(open('gpurun_out/bench4.json'))
print(d['value'], d['ms_per_step'], json.dumps(d['roofline'], indent=1), d['autotune']['best'], d['clocks'])
"
