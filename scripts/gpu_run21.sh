timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "graph or split_pieces or cofactoring or shard" 2>&1 | grep -E "Error|assert|FAILED|passed|failed" | head -20
