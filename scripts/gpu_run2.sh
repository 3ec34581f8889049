set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 2000 --durations=8 2>&1 | tail -25
timeout 600 python bench.py --steps 3 --warmup 3 --cpu-seconds 10 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; tail -3 gpurun_out/bench2.err; cat gpurun_out/bench2.json
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python scripts/profile_kernel.py c5 34 2 > gpurun_out/plain_prof.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -c 2 -o gpurun_out/prof_c5 \
  python scripts/profile_kernel.py c5 34 2 > gpurun_out/ncu_prof.log 2>&1
tail -2 gpurun_out/ncu_prof.log; ls -la gpurun_out
