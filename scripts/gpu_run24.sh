mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/bench24_torchrun.json 2> gpurun_out/bench24_torchrun.err; tail -2 gpurun_out/bench24_torchrun.err
python -c "
import json; d=json.load(open('gpurun_out/bench24_torchrun.json'))
print(d['value'], d['ms_per_step'], d['count'], d['gpu_launches'], d['roofline']['frac'], d['e2e']['value'], d['jit_prep_s'], d['cpu_baseline'])
"
