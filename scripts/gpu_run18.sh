mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q --timeout 2400 --durations=5 2>&1 | tail -10
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
