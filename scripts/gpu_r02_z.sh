#!/bin/bash
# the slot-14 C4 preset: its parity tests, smoke, the bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/z_smoke.log
timeout 1200 python -m pytest tests -x -q -m gpu -k "exhaustive_bench or imad_pair or c4 or multi_rank or ranges or count_shard or rows or enumerate" > gpurun_out/z_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/z_pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/z_bench.json 2> gpurun_out/z_bench.err
echo "rc=$?" >> gpurun_out/z_bench.err
