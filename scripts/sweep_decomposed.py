"""Decomposed-plan frontier on one GPU: for each configuration, the cold
preparation time (decomposition + role searches + PTX compile, persistent JIT
cache off) and the median replay step (CUDA events), plus the count.  One JSON
line per configuration.  Usage: python scripts/sweep_decomposed.py '[{"split_pieces": 4096}, ...]'"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402
from paper_1310_6978_b200 import presets  # noqa: E402


def main():
    cfgs = json.loads(sys.argv[1])
    name = sys.argv[2] if len(sys.argv) > 2 else "c5"
    text, n, _ = W.config(name)
    torch.cuda.set_device(0)
    st = torch.cuda.current_stream()
    ref = None
    for extra in cfgs:
        p = presets.apply(bfa.Program(text), presets.DECOMPOSED, jit_cache=0, **extra)
        c = torch.zeros(1, dtype=torch.int64, device="cuda")
        t0 = time.perf_counter()
        p.count_range(n, 0, 1 << n, out=c, stream=st)
        torch.cuda.synchronize()
        prep = time.perf_counter() - t0
        for _ in range(3):
            p.count_range(n, 0, 1 << n, out=c, stream=st)
        torch.cuda.synchronize()
        ll = bfa.last_launch()
        ms = []
        for _ in range(7):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            p.count_range(n, 0, 1 << n, out=c, stream=st)
            b.record(st)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        cnt = int(c.item())
        ref = cnt if ref is None else ref
        print(json.dumps({"cfg": extra, "prep_s": prep, "ms": statistics.median(ms), "count": cnt, "same": cnt == ref,
                          "kernels": ll.get("kernels"), "queue": ll.get("queue"), "decompose_s": ll.get("decompose_s"),
                          "cells_lop3": ll.get("cells_lop3"), "cells_imad": ll.get("cells_imad")}), flush=True)


if __name__ == "__main__":
    main()
