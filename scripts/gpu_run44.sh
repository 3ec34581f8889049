timeout 900 python -m pytest tests/test_gpu_parity.py -x -q --timeout 800 -k "work_queue" 2>&1 | grep -E "Error|error|assert|^E " | head -20
