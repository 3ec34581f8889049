export BFA_JIT_CACHE=/tmp/bfa_cold_$$
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1000 -k "work_queue or split_pieces or shard" 2>&1 | tail -2
export BFA_JIT_CACHE=/tmp/bfa_cold2_$$
t0=$(date +%s)
timeout 1500 python bench.py > gpurun_out/q4_bench.json 2> gpurun_out/q4_bench.err; tail -3 gpurun_out/q4_bench.err
echo "bench wall $(( $(date +%s) - t0 )) s"
python -c "
import json; d=json.load(open('gpurun_out/q4_bench.json'))
print({k: d[k] for k in ('value','ms_per_step','count','gpu_launches','jit_prep_s')}, d['roofline']['frac'], d['e2e']['value'], d['clocks'])
print(d['autotune']['best']); print(d['autotune'].get('partial_evaluation'))
"
