mkdir -p gpurun_out
for ic in 50 35; do
OPTS="slot_bits=5,imad_cost_pct=$ic"
python scripts/profile_kernel.py c5 42 1 $OPTS > gpurun_out/plain_prof3_$ic.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -c 1 -o gpurun_out/prof3_c5_$ic \
  python scripts/profile_kernel.py c5 42 1 $OPTS > gpurun_out/ncu_prof3_$ic.log 2>&1
tail -1 gpurun_out/ncu_prof3_$ic.log
done
