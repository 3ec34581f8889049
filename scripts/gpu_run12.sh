mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "geometries or paper_scale or edge or ranges" 2>&1 | tail -4
timeout 900 python bench.py --config paper_2p17 --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench12_p17.json 2> gpurun_out/bench12_p17.err; tail -3 gpurun_out/bench12_p17.err
python -c "
import json; d=json.load(open('gpurun_out/bench12_p17.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['launch'], d['cpu_baseline'])
"
