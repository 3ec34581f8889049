set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc; lscpu | grep "Model name"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q -k "not full_set_bits" --timeout 900 2>&1 | tail -30
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 5 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; tail -3 gpurun_out/bench1.err; cat gpurun_out/bench1.json
