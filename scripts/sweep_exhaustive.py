"""Exhaustive-kernel variants on one GPU: cold preparation and median full-cube
count time (CUDA events) per option set, with the count.  One JSON line each.
    python scripts/sweep_exhaustive.py c5 '[{"slot_bits": 6, "inner_bits": 3}, ...]'"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402
from paper_1310_6978_b200 import presets  # noqa: E402

cfg = sys.argv[1]
text, n, _ = W.config(cfg)
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
for extra in json.loads(sys.argv[2]):
    p = presets.apply(bfa.Program(text), presets.exhaustive(cfg), jit_cache=0, **extra)
    c = torch.zeros(1, dtype=torch.int64, device="cuda")
    t0 = time.perf_counter()
    p.count_range(n, 0, 1 << n, out=c, stream=st)
    torch.cuda.synchronize()
    prep = time.perf_counter() - t0
    ms = []
    for _ in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        p.count_range(n, 0, 1 << n, out=c, stream=st)
        b.record(st)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    ll = bfa.last_launch()
    seg = ll["segments"][0]
    words = 1 << (n - 5)
    print(json.dumps({"cfg": cfg, "opts": extra, "prep_s": prep, "ms": statistics.median(ms), "count": int(c.item()),
                      "cells_per_word": (ll["cells_lop3"] + ll["cells_imad"]) / words,
                      "lop3_per_word": ll["cells_lop3"] / words, "regs": seg["regs"],
                      "blocks_per_sm": seg["blocks_per_sm"]}), flush=True)
