mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; tail -c 200 gpurun_out/fc_smoke.log; echo
timeout 2700 python -m pytest tests -x -q -m gpu --timeout 2400 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; tail -2 gpurun_out/fc_bench.err
python -c "
import json; d=json.load(open('gpurun_out/fc_bench.json'))
print({k: d[k] for k in ('value','ms_per_step','count','gpu_launches','jit_prep_s','executed_valuations_per_s')}, d['roofline']['frac'], d['e2e']['value'], d['clocks'])
"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fc_ref.json 2>&1; head -c 300 gpurun_out/fc_ref.json
