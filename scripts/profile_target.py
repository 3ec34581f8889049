"""Profiling targets for ncu (one GPU): the bench's kernels, launched as the
bench launches them, `steps` times (ncu -s/-c pick the launches).

    python scripts/profile_target.py exhaustive|c4_exhaustive|replay|materialised|c4_eval [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402
from paper_1310_6978_b200 import presets  # noqa: E402

what = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
torch.cuda.set_device(0)
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
if what in ("exhaustive", "c4_exhaustive", "replay"):
    text, n, _ = W.config("c4" if what == "c4_exhaustive" else "c5")
    preset = presets.DECOMPOSED if what == "replay" else presets.exhaustive("c4" if what == "c4_exhaustive" else "c5")
    p = presets.apply(bfa.Program(text), preset)
    for _ in range(steps):
        p.count_range(n, 0, 1 << n, out=cnt)
    torch.cuda.synchronize()
    print(what, int(cnt.item()), bfa.last_launch())
elif what == "c4_eval":
    text, n, _ = W.config("c4")
    p = presets.apply(bfa.Program(text), presets.exhaustive("c4"))
    vec = torch.empty(bfa.words_for(n), dtype=torch.int64, device="cuda")
    for _ in range(steps):
        p.eval_range(n, 0, 1 << n, out=vec, count_out=cnt)
    torch.cuda.synchronize()
    print(what, int(cnt.item()), bfa.last_launch())
elif what == "materialised":
    for cfg in ("c2", "c2_n32"):
        text, n, _ = W.config(cfg)
        p = bfa.Program(text)
        out = torch.empty(bfa.words_for(n), dtype=torch.int64, device="cuda")
        for variant in (0, 1):
            for _ in range(steps):
                p.eval_materialised(n, variant, out=out, count_out=cnt)
            torch.cuda.synchronize()
            print(cfg, variant, int(cnt.item()), bfa.last_launch())
        del out
        torch.cuda.empty_cache()
else:
    raise SystemExit(f"unknown target {what}")
