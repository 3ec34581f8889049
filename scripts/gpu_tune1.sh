set -x
mkdir -p gpurun_out
python scripts/tune.py c5 38 "dual_pipe=0" "imad_cost_pct=20" "imad_cost_pct=35" "imad_cost_pct=50" "imad_cost_pct=60" "imad_cost_pct=35,slot_bits=1" "imad_cost_pct=35,slot_bits=3" "imad_cost_pct=35,thread_bits=7" "dual_pipe=0,slot_bits=3" "dual_pipe=0,slot_bits=1" 2>&1 | tee gpurun_out/tune_c5.log
python scripts/tune.py c4 36 "dual_pipe=0" "imad_cost_pct=20" "imad_cost_pct=35" "imad_cost_pct=50" "imad_cost_pct=60" "imad_cost_pct=35,slot_bits=3" "imad_cost_pct=35,inner_bits=6" "dual_pipe=0,inner_bits=6" 2>&1 | tee gpurun_out/tune_c4.log
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "geometries or random_terms or edge or ranges" 2>&1 | tail -5
