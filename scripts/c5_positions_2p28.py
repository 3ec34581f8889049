"""Evidence beyond the pytest sizes (SURVEY P-13 asks for 2^28 C5 sub-cubes):
the exact headline kernel (presets.exhaustive("c5")) against the CPU oracle on
4 random 2^28-position ranges of its enumeration order.

    python scripts/c5_positions_2p28.py oracle  out.json   # CPU only (~10 min per range on 8 cores)
    python scripts/c5_positions_2p28.py gpu     out.json   # the kernel's counts for the same ranges

The oracle side counts the renamed program f'(x) = f(x renamed v -> perm[v])
over contiguous valuation ranges (perm from bfa_roles, host only, for a
148-SM B200); the GPU side runs bfa_count_positions on the same ranges."""
import json
import os
import re
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402
from paper_1310_6978_b200 import presets  # noqa: E402

mode, path = sys.argv[1], sys.argv[2]
text, n, _ = W.config("c5")
p = presets.apply(bfa.Program(text), presets.exhaustive("c5"))
perm = p.roles(n, n, sms=148)
rng = np.random.default_rng(20261019)
ranges = [int(rng.integers(0, 1 << (n - 28))) << 28 for _ in range(4)]
if mode == "oracle":
    import oracle
    text2 = re.sub(r"\bx(\d+)\b", lambda m: f"x{perm[int(m.group(1))]}", text)
    res = []
    for lo in ranges:
        t0 = time.time()
        c = oracle.count(text2, n, lo, lo + (1 << 28))
        res.append({"lo": lo, "hi": lo + (1 << 28), "oracle": c, "seconds": time.time() - t0})
        print(res[-1], flush=True)
    json.dump({"perm": perm, "preset": presets.exhaustive("c5"), "ranges": res}, open(path, "w"), indent=1)
else:
    import torch
    ref = json.load(open(path))
    assert ref["perm"] == perm, "role permutation differs from the oracle run's"
    out = []
    for r in ref["ranges"]:
        g = int(p.count_positions(n, n, r["lo"], r["hi"]).item())
        torch.cuda.synchronize()
        out.append(dict(r, gpu=g, equal=g == r["oracle"]))
        print(out[-1], flush=True)
    json.dump({"perm": perm, "preset": presets.exhaustive("c5"), "ranges": out,
               "all_equal": all(x["equal"] for x in out)}, open(path.replace(".json", "_gpu.json"), "w"), indent=1)
