"""Builds the in-tree C-ABI library ``liblobra.so`` with nvcc for sm_100a.

    python -m paper_2509_01193_b200.build

Sources: ``csrc/*.cu`` (kernels + host entry points) and ``csrc/*.cpp`` (dispatch, NCCL
plumbing).  cudart is linked statically; NCCL is dlopen'ed at run time (the copy torch
loads), so the library has no link-time dependency on either torch or NCCL.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "liblobra.so")


def _nccl_include() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for p in spec.submodule_search_locations:
            cands.append(os.path.join(p, "nccl", "include"))
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (nvidia-nccl wheel)")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def build(verbose: bool = False, force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) +
                  glob.glob(os.path.join(HERE, "csrc", "*.cpp")))
    deps = srcs + glob.glob(os.path.join(HERE, "csrc", "*.h")) + \
        glob.glob(os.path.join(HERE, "csrc", "*.cuh")) + [os.path.join(ROOT, "include", "lobra.h")]
    if not force and os.path.exists(LIB):
        lt = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= lt for d in deps):
            return LIB
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
           "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", LIB + ".tmp"] + srcs + ["-ldl", "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building liblobra.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
