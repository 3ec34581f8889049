mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "batch" 2>&1 | tail -4
