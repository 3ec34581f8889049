mkdir -p gpurun_out
OPTS=$(cat gpurun_out/best20.json 2>/dev/null || echo '{"slot_bits": 5, "inner_bits": 4, "imad_cost_pct": 50, "dual_pipe": 1, "min_blocks": 0, "thread_bits": 8, "kernel_cofactor_bits": 5, "split_pieces": 16}')
echo "$OPTS"
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/plain22.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -s 1700 -c 4 -o gpurun_out/prof22 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --options "$OPTS" > gpurun_out/ncu22.log 2>&1
tail -2 gpurun_out/ncu22.log
