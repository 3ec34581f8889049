"""Build libbfa.so in-tree (sm_100a).  Usable without a GPU (nvcc and NVRTC
cross-compile).  Invoked by __graft_entry__.build() and on import if the
library is missing.

    nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3   bfa_kernels.cu
    g++  -O2 -std=c++17 -fvisibility=hidden                      bfa_compiler.cpp bfa_runtime.cpp
    link: cudart, NVRTC, nvrtc-builtins and nvptxcompiler STATIC, so the JIT
          never binds to another NVRTC already loaded in the process (torch).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(HERE, "libbfa.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = {
    "bfa_kernels.cu": [NVCC, *ARCH, "-lineinfo", "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-c"],
    "bfa_compiler.cpp": ["g++", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-std=c++17", "-Wall", "-Wextra",
                         f"-I{CUDA}/include", "-c"],
    "bfa_runtime.cpp": ["g++", "-O2", "-g", "-fPIC", "-fvisibility=hidden", "-std=c++17", "-Wall", "-Wextra",
                        f"-I{CUDA}/include", "-c"],
}
HEADERS = ["bfa_compiler.hpp", "bfa_kernels.hpp", os.path.join("..", "..", "include", "bfa.h")]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdr_t = max(_mtime(os.path.join(CSRC, h)) for h in HEADERS)
    jobs = []
    objs = []
    for src, cmd in SOURCES.items():
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            jobs.append(cmd + [s, "-o", o])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)

    with ThreadPoolExecutor(max_workers=3) as ex:
        list(ex.map(run, jobs))
    if jobs or force or _mtime(LIB) < max(_mtime(o) for o in objs):
        link = ["g++", "-shared", "-o", LIB + ".tmp", *objs, f"-L{CUDA}/lib64",
                "-Wl,--start-group", "-lcudart_static", "-lnvrtc_static", "-lnvrtc-builtins_static",
                "-lnvptxcompiler_static", "-Wl,--end-group", "-lpthread", "-ldl", "-lrt",
                "-Wl,--exclude-libs,ALL", "-Wl,--no-undefined", "-s"]
        run(link)
        os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
