#!/bin/bash
# End-of-round check on one B200: smoke, the full -m gpu suite, the default
# bench line and the reference arm (as the driver runs them).
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fc_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fc_smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/fc_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/fc_pytest.log
timeout 1200 python bench.py > gpurun_out/fc_bench.json 2> gpurun_out/fc_bench.err; echo "bench rc=$?" >> gpurun_out/fc_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fc_ref.json 2> gpurun_out/fc_ref.err
