mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --timeout 2000 --durations=6 2>&1 | tail -14
