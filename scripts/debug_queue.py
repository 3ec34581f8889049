"""Debug: C5 decomposed counts (32768 leaves) over several fresh compiles and replays."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1310_6978_b200 as bfa, workloads as W
from paper_1310_6978_b200 import presets
text, n, _ = W.config("c5")
extra = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
p = presets.apply(bfa.Program(text), presets.DECOMPOSED, jit_cache=0, **extra)
c = torch.zeros(1, dtype=torch.int64, device="cuda")
t = time.time()
res = []
for i in range(6):
    p.count_range(n, 0, 1 << n, out=c)
    torch.cuda.synchronize()
    res.append(int(c.item()))
    if i == 0:
        prep = time.time() - t
q = p.count(n)
print(json.dumps({"extra": extra, "env": os.environ.get("BFA_PTX_SERIAL"), "prep": prep, "counts": res, "count": q,
                  "ok": all(x == 1469173439442 for x in res + [q])}), flush=True)
