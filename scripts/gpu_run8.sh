mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "geometries" 2>&1 | tail -3
python scripts/tune.py c5 34 "engine=1" "dual_pipe=0" "slot_bits=5,imad_cost_pct=35" 2>&1 | tee gpurun_out/ablation_c5.log
python scripts/tune.py c4 32 "engine=1" "dual_pipe=0" "slot_bits=5,imad_cost_pct=50" 2>&1 | tee gpurun_out/ablation_c4.log
