mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q --timeout 1200 -k "count_shard" 2>&1 | tail -4
python - <<'PY'
import sys, time, torch
sys.path.insert(0, ".")
import paper_1310_6978_b200 as bfa, workloads as W
text, n, _ = W.config("c5")
p = bfa.Program(text); p.autotune(n)
for world in (2, 4, 8):
    ts = []
    for r in range(world):
        p.count_shard(n, r, world); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); p.count_shard(n, r, world); e.record(); torch.cuda.synchronize()
        ts.append(round(s.elapsed_time(e), 2))
    print("world", world, "per-rank ms", ts, "load", bfa.last_launch()["load"])
PY
