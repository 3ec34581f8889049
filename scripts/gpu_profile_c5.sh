# work-queue kernels of the autotuned C5 configuration (32768 leaves, 71 modules per step), replayed via --options
mkdir -p gpurun_out
O='{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "min_blocks": 0, "thread_bits": 8, "kernel_cofactor_bits": 0, "split_pieces": 32768, "queue_bodies": 512}'
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --options "$O" > gpurun_out/p7_bench.json 2> gpurun_out/p7_bench.err || { tail -5 gpurun_out/p7_bench.err; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__registers_per_thread --clock-control none -k regex:bfa_kernel -c 3000 --csv \
  --log-file gpurun_out/p7_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --options "$O" > gpurun_out/p7_ncu.log 2>&1
tail -1 gpurun_out/p7_ncu.log
timeout 1000 ncu --set full --clock-control none -k regex:bfa_kernel -s 142 -c 71 -o gpurun_out/p7_full \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --options "$O" > gpurun_out/p7_full.log 2>&1
tail -1 gpurun_out/p7_full.log
ncu -i gpurun_out/p7_full.ncu-rep --page raw --csv > gpurun_out/p7_full_raw.csv 2>/dev/null
rm -f gpurun_out/p7_full.ncu-rep
ls -la gpurun_out/p7_*
