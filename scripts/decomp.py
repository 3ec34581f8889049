"""Time full-cube counts over (split_pieces, kernel_cofactor_bits) settings (GPU)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1]
text, n, _ = W.config(cfg)
base = json.loads(sys.argv[2])
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
ref = None
for spec in sys.argv[3:]:
    sp, j = (int(x) for x in spec.split(","))
    p = bfa.Program(text)
    for k, v in base.items():
        p.set_option(k, v)
    p.set_option("split_pieces", sp).set_option("kernel_cofactor_bits", j)
    t0 = time.time()
    p.count_range(n, 0, 1 << n, out=cnt)
    torch.cuda.synchronize()
    prep = time.time() - t0
    for _ in range(2):
        p.count_range(n, 0, 1 << n, out=cnt)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5):
        p.count_range(n, 0, 1 << n, out=cnt)
    e.record()
    torch.cuda.synchronize()
    c = int(cnt.item())
    ref = c if ref is None else ref
    ll = bfa.last_launch()
    l3, im = ll.get("cells_lop3", 0), ll.get("cells_imad", 0)
    floor = max(l3 / 18.6e12, (l3 + im) / 35.2e12) * 1e3   # ALU-pipe / issue bound, ms
    print(json.dumps({"sp": sp, "j": j, "ms": round(s.elapsed_time(e) / 5, 3), "ok": c == ref, "prep_s": round(prep, 1),
                      "count": c, "decided": ll.get("valuations_decided"), "kernels": ll.get("kernels"),
                      "cells_lop3": l3, "cells_imad": im, "alu_floor_ms": round(floor, 3),
                      "decompose_s": ll.get("decompose_s"), "queue": ll.get("queue")}), flush=True)
