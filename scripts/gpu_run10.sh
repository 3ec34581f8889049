mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; tail -3 gpurun_out/bench10.err
python -c "
import json; d=json.load(open('gpurun_out/bench10.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'])
for c in sorted(d['autotune']['candidates'], key=lambda c: c['ms'])[:6]: print(c)
"
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench10_c4.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/bench10_c4.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'])
"
