mkdir -p gpurun_out
OPTS="slot_bits=5,imad_cost_pct=35"
python scripts/profile_kernel.py c5 34 2 $OPTS > gpurun_out/plain_prof2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -c 1 -o gpurun_out/prof2_c5 \
  python scripts/profile_kernel.py c5 34 2 $OPTS > gpurun_out/ncu_prof2.log 2>&1
OPTS4="slot_bits=5,imad_cost_pct=50"
python scripts/profile_kernel.py c4 36 2 $OPTS4 > gpurun_out/plain_prof2c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:bfa_kernel -c 1 -o gpurun_out/prof2_c4 \
  python scripts/profile_kernel.py c4 36 2 $OPTS4 > gpurun_out/ncu_prof2c4.log 2>&1
tail -2 gpurun_out/ncu_prof2.log gpurun_out/ncu_prof2c4.log
