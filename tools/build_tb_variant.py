"""Build a variant of the library with another two-step-kernel tiling (tools only).

python tools/build_tb_variant.py HT PF [EARLY [NAME=VALUE ...]]  ->  paper_1703_00186_b200/variants/liblb_ht<HT>_pf<PF>[_e1].so
(lb_tb.cu compiled with -DLB_TB_HT=HT -DLB_TB_PF=PF, linked with the default
build's other objects).  Load it with LB_D2Q37_LIB=<path>.  PF = 0: one
state-n buffer refilled right after the phase-1 gather; EARLY = 1: the PF + 1
buffers refilled that way (loads NB iterations ahead).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1703_00186_b200 import _build  # noqa: E402


def main():
    ht, pf = int(sys.argv[1]), int(sys.argv[2])
    early = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    extra = sys.argv[4:]  # further NAME=VALUE defines, e.g. LB_TB_DECOUPLE=1
    tag = os.environ.get("TB_TAG", "") + f"ht{ht}_pf{pf}" + (f"_e{early}" if early else "") + "".join(
        "_" + d.split("=")[0].replace("LB_TB_", "").lower() + d.split("=")[1] for d in extra)
    _build.build()
    nd = _build.nccl_dir()
    out = os.path.join(_build.HERE, "variants")
    os.makedirs(out, exist_ok=True)
    obj = os.path.join(out, f"lb_tb_{tag}.o")
    flags = [_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "--expt-relaxed-constexpr",
             "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math", "-Xptxas", "-v,-warn-spills",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(_build.HERE, "csrc"), "-I", os.path.join(nd, "include"),
             f"-DLB_TB_HT={ht}", f"-DLB_TB_PF={pf}", f"-DLB_TB_EARLY={early}", *("-D" + d for d in extra)]
    src = os.environ.get("TB_SRC") or os.path.join(_build.HERE, "csrc", "lb_tb.cu")  # TB_SRC: e.g. an older revision
    r = subprocess.run(["nvcc", *flags, "-c", src, "-o", obj], capture_output=True, text=True)
    sys.stdout.write("\n".join(l for l in (r.stdout + r.stderr).splitlines()
                               if "k_step2_tb" in l or "registers" in l or "spill" in l or "error" in l))
    if r.returncode:
        sys.exit(r.returncode)
    objdir = os.path.join(_build.HERE, "build_obj")
    objs = [os.path.join(objdir, f) for f in sorted(os.listdir(objdir)) if f.endswith(".o") and f != "lb_tb.cu.o"]
    so = os.path.join(out, f"liblb_{tag}.so")
    r = subprocess.run(["nvcc", _build.ARCH, "-shared", obj, *objs, "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
                        "-Xlinker", "-rpath," + os.path.join(nd, "lib"), "-o", so], capture_output=True, text=True)
    print(r.stdout + r.stderr)
    if r.returncode:
        sys.exit(r.returncode)
    print(so)


if __name__ == "__main__":
    main()
