OPTS='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "min_blocks": 0, "thread_bits": 8, "kernel_cofactor_bits": 4, "split_pieces": 128}'
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/plain28.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches28.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/ncu28.log 2>&1
grep -o '"ms_per_step": [0-9.]*' gpurun_out/plain28.log
