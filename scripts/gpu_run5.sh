mkdir -p gpurun_out
python - <<'PY'
import json, torch, sys
sys.path.insert(0, ".")
import paper_1310_6978_b200 as bfa, workloads as W
for cfg in ("c5", "c4", "c3_posets"):
    text, n, _ = W.config(cfg)
    p = bfa.Program(text)
    rep = p.autotune(n)
    print(cfg, "best", rep["best"])
    for c in sorted(rep["candidates"], key=lambda c: c["ms"])[:8]:
        print("   ", c)
PY
