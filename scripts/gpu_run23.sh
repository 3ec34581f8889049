mkdir -p gpurun_out
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_posets3 or generators or edge_cases or ranges_concatenate or materialised_modes or enumerate_matches or batch_counts" 2>&1 | tail -6
