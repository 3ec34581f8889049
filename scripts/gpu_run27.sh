rm -rf /root/.cache/bfa_jit
for i in 1 2; do
timeout 1200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench27_$i.json 2> gpurun_out/bench27_$i.err; tail -2 gpurun_out/bench27_$i.err
python -c "
import json; d=json.load(open('gpurun_out/bench27_$i.json'))
print({k: d[k] for k in ('value','ms_per_step','count','gpu_launches','jit_prep_s','executed_valuations_per_s')}, d['roofline']['frac'], d['autotune']['best'], d['autotune']['kernel_cofactoring'])
"
done
du -sh /root/.cache/bfa_jit
