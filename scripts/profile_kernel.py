"""Launch the bench's register-mode count kernel on a sub-range of a config
(same JIT variant and launch geometry as bench.py), for ncu captures.

    python scripts/profile_kernel.py [config] [log2_valuations] [launches] [opt=v,opt=v]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 36
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 3
text, n, _ = W.config(cfg)
p = bfa.Program(text)
for kv in filter(None, (sys.argv[4] if len(sys.argv) > 4 else "").split(",")):
    a, b = kv.split("=")
    p.set_option(a, int(b))
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
lo = (1 << n) - (1 << k)
for _ in range(launches):
    p.count_range(n, lo, 1 << n, out=cnt)
torch.cuda.synchronize()
print(cfg, n, k, int(cnt.item()), bfa.last_launch())
