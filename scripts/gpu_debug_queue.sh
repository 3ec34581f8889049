cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/debug_queue.py '{}' >> gpurun_out/dbg2.jsonl 2>&1
BFA_PTX_BRX=1 python scripts/debug_queue.py '{"queue_bodies": 256}' >> gpurun_out/dbg2.jsonl 2>&1
