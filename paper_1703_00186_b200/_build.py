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
    flags = [ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "--expt-relaxed-constexpr",
             "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
             "-Xptxas", "-v,-warn-spills",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include")]
    objdir = os.path.join(HERE, "build_obj")
    os.makedirs(objdir, exist_ok=True)
    # one nvcc per translation unit, in parallel (lb_kernels.cu and lb_tb.cu
    # each take minutes), then one link
    procs, objs = [], []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [nvcc, *flags, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)))
    log_txt, failed = [], False
    for cmd, pr in procs:
        out, _ = pr.communicate()
        log_txt.append(" ".join(cmd) + "\n" + out)
        failed |= pr.returncode != 0
    link = [nvcc, ARCH, "-shared", *objs, "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath," + os.path.join(nd, "lib"), "-o", SO + ".tmp"]
    if not failed:
        r = subprocess.run(link, capture_output=True, text=True)
        log_txt.append(" ".join(link) + "\n" + r.stdout + r.stderr)
        failed = r.returncode != 0
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as fh:
        fh.write("\n".join(log_txt))
    if failed:
        sys.stderr.write("\n".join(log_txt))
        raise RuntimeError("nvcc failed (see %s)" % log)
    if verbose:
        sys.stderr.write("\n".join(log_txt))
    os.replace(SO + ".tmp", SO)
    return SO


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(SO)
