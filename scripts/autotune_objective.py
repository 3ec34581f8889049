"""bfa_autotune's total-cost objective on C5: the plan chosen for
tune_counts = 1 (one cold count) and for many counts, with every plan tried
(preparation, step, total) or skipped (predicted preparation)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402
from paper_1310_6978_b200 import presets  # noqa: E402

text, n, _ = W.config("c5")
torch.cuda.set_device(0)
for k in [int(x) for x in sys.argv[1:]] or [1, 100000]:
    p = presets.apply(bfa.Program(text), presets.cold("c5"), jit_cache=0, tune_counts=k)
    t0 = time.perf_counter()
    rep = p.autotune(n)
    dt = time.perf_counter() - t0
    c = p.count(n)
    print(json.dumps({"tune_counts": k, "autotune_s": dt, "count": c, "best": rep["best"], "plans": rep["plans"]}),
          flush=True)
