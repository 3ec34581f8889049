"""Time the register-mode count kernel over option settings (GPU).
    python scripts/tune.py <config> <log2_range> "<opt=v,opt=v>" ["..."]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402

cfg, k = sys.argv[1], int(sys.argv[2])
text, n, _ = W.config(cfg)
lo, hi = (1 << n) - (1 << k), 1 << n
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ref = None
for spec in sys.argv[3:]:
    p = bfa.Program(text)
    for kv in filter(None, spec.split(",")):
        a, b = kv.split("=")
        p.set_option(a, int(b))
    t0 = time.time()
    p.count_range(n, lo, hi, out=cnt)
    torch.cuda.synchronize()
    jit = time.time() - t0
    c = int(cnt.item())
    if ref is None:
        ref = c
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    s.record()
    for _ in range(reps):
        p.count_range(n, lo, hi, out=cnt)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / reps
    ll = bfa.last_launch()
    L = ll.get("segments") or [{"words": 0, "regs": None, "blocks_per_sm": None, "luts_inner": ll.get("ops"),
                                "imads_inner": 0, "derived_inner": 0, "imad_cost": None}]
    g = max(L, key=lambda x: x["words"])
    print(json.dumps({"cfg": cfg, "opts": spec, "ms": round(ms, 3), "Gval_per_s": round((hi - lo) / ms / 1e6, 1),
                      "ok": c == ref, "count": c, "jit_s": round(jit, 2), "regs": g["regs"], "bps": g["blocks_per_sm"],
                      "luts_inner": g["luts_inner"], "imads_inner": g["imads_inner"],
                      "derived_inner": g["derived_inner"], "imad_cost": g["imad_cost"]}), flush=True)
