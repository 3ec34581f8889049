mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "split_pieces or count_shard or cofactoring" 2>&1 | tail -4
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 > gpurun_out/bench17.json 2> gpurun_out/bench17.err; tail -3 gpurun_out/bench17.err
python -c "
import json; d=json.load(open('gpurun_out/bench17.json'))
print(d['value'], d['ms_per_step'], d['count'], d['roofline']['frac'], d['roofline']['per_unit'], d['autotune']['best'], d['autotune'].get('kernel_cofactoring'), d['jit_prep_s'], d['decided_at_compile_time'], d['executed_valuations_per_s'])
"
