timeout 1200 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench26.json 2> gpurun_out/bench26.err; tail -2 gpurun_out/bench26.err
python -c "
import json; d=json.load(open('gpurun_out/bench26.json'))
print({k: d[k] for k in ('value','ms_per_step','count','gpu_launches','jit_prep_s','executed_valuations_per_s')}, d['roofline']['frac'], d['autotune']['best'], d['autotune']['kernel_cofactoring'])
json.dump(d['autotune']['best'], open('gpurun_out/best26.json','w'))
"
