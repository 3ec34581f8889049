"""SASS instruction mix of a generated kernel (CPU-only: NVRTC + cuobjdump).
    python scripts/sass_mix.py <config> [what=1] [opt=value ...]"""
import collections
import os
import re
import subprocess
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_6978_b200 as bfa  # noqa: E402
import workloads as W  # noqa: E402


def mix(prog, what=1):
    cub = prog.jit_cubin(what)
    with tempfile.NamedTemporaryFile(suffix=".cubin") as f:
        f.write(cub)
        f.flush()
        sass = subprocess.run(["cuobjdump", "-sass", f.name], capture_output=True, text=True).stdout
        res = subprocess.run(["cuobjdump", "-res-usage", f.name], capture_output=True, text=True).stdout
    ops = [m.group(1) for m in re.finditer(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", sass)]
    regs = re.search(r"REG:(\d+)", res).group(1)
    local = re.search(r"LOCAL:(\d+)", res).group(1)
    return collections.Counter(ops), int(regs), int(local)


if __name__ == "__main__":
    cfg = sys.argv[1]
    what = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    text, n, _ = W.config(cfg)
    p = bfa.Program(text)
    for kv in sys.argv[3:]:
        k, v = kv.split("=")
        p.set_option(k, int(v))
    c, regs, local = mix(p, what)
    print(cfg, "regs", regs, "local", local, c.most_common(14))
