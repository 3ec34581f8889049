"""Kernel-level cofactoring sweep (GPU): autotune, then time counts with
kernel_cofactor_bits = j."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1]
js = [int(x) for x in sys.argv[2].split(",")]
text, n, expect = W.config(cfg)
p = bfa.Program(text)
t0 = time.time()
tune = p.autotune(n)
print("autotune", tune["best"], round(time.time() - t0, 1), "s", flush=True)
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ref = None
for j in js:
    p.set_option("kernel_cofactor_bits", j)
    t0 = time.time()
    p.count_range(n, 0, 1 << n, out=cnt)
    torch.cuda.synchronize()
    prep = time.time() - t0
    c = int(cnt.item())
    ref = c if ref is None else ref
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        p.count_range(n, 0, 1 << n, out=cnt)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 3
    ll = bfa.last_launch()
    print(json.dumps({"cfg": cfg, "j": j, "ms": round(ms, 3), "val_per_s": (1 << n) / ms * 1e3, "count": c,
                      "ok": c == ref and (expect is None or c == expect), "prep_s": round(prep, 1),
                      "kernels": ll.get("kernels")}), flush=True)
