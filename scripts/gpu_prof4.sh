# launch list of the autotuned C5 bench configuration (replayed via --options)
mkdir -p gpurun_out
O='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "min_blocks": 0, "thread_bits": 8, "kernel_cofactor_bits": 4, "split_pieces": 128}'
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$O" > gpurun_out/p4_bench.json 2> gpurun_out/p4_bench.err || exit 1
timeout 1800 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:bfa_kernel -c 9000 --csv \
  --log-file gpurun_out/p4_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --options "$O" > gpurun_out/p4_ncu.log 2>&1
tail -3 gpurun_out/p4_ncu.log
