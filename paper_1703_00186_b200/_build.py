"""Build liblb_d2q37.so (the C-ABI CUDA library) in-tree for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a, -lineinfo, --fmad=false (all
contractions in the kernels are explicit __fma_rn), host code with
-ffp-contract=off (K_wall must be bit-identical to the canonical tree, G16),
linked against the NCCL that ships with the torch wheel (one NCCL in-process).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "liblb_d2q37.so")
ARCH = "-gencode=arch=compute_100a,code=sm_100a"


def nccl_dir() -> str:
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in list(spec.submodule_search_locations or []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers from the torch wheel (nvidia/nccl) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "lb.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    nd = nccl_dir()
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "--expt-relaxed-constexpr",
           "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
           "-Xptxas", "-v,-warn-spills",
           "-shared", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
           *sources(),
           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
           "-Xlinker", "-rpath," + os.path.join(nd, "lib"),
           "-o", SO + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed (see %s)" % log)
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
