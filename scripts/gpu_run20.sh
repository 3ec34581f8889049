mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "graph or split_pieces or cofactoring or shard" 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench20.json 2> gpurun_out/bench20.err; tail -3 gpurun_out/bench20.err
python -c "
import json; d=json.load(open('gpurun_out/bench20.json'))
print(d['value'], d['ms_per_step'], d['count'], d['gpu_launches'], d['roofline']['frac'], d['autotune']['best'], d['jit_prep_s'], d['executed_valuations_per_s'])
json.dump(d['autotune']['best'], open('gpurun_out/best20.json','w'))
"
OPTS=$(cat gpurun_out/best20.json)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/plain20.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches20.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/ncu20.log 2>&1
grep -o '"ms_per_step": [0-9.]*' gpurun_out/plain20.log
