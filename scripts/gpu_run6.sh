mkdir -p gpurun_out
for c in c2 c2_fused c2_n32 c2_n32_fused; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/bench6_$c.json 2> gpurun_out/bench6_$c.err; tail -2 gpurun_out/bench6_$c.err
  python -c "
import json; d=json.load(open('gpurun_out/bench6_$c.json'))
print('$c', round(d['value']/1e9,2), 'Gval/s', round(d['ms_per_step'],2), 'ms', 'count', d['count'], 'GB/s', round(d['roofline']['achieved'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), d['launch'])
"
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_torchrun.json 2> gpurun_out/bench6_torchrun.err; tail -3 gpurun_out/bench6_torchrun.err; head -c 400 gpurun_out/bench6_torchrun.json
