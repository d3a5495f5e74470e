"""SASS census of the built library (measurement tool; no GPU needed).

    python tools/sass_census.py [--so PATH] [--out profiles/r02_sass.json]

Disassembles liblb_d2q37.so with cuobjdump -sass and counts, per kernel
(demangled, grouped by template instantiation), the instructions that show
how the hot path maps to sm_100a: TMA loads (UTMALDG), mbarrier / async
sync (SYNCS), FP64 arithmetic (DFMA / DADD / DMUL), shared and global memory
(LDS / STS / LDG / STG) and local memory (LDL / STL: spills — must be zero in
every hot kernel).  Static counts (instructions in the binary), not dynamic.
"""
from __future__ import annotations

import argparse
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1703_00186_b200", "liblb_d2q37.so")
OPS = ["UTMALDG", "UTMASTG", "UBLKCP", "SYNCS", "DFMA", "DADD", "DMUL", "MUFU", "LDS", "STS", "LDG", "STG",
       "LDL", "STL", "BAR", "SHFL", "UMOV"]
HOT = ("k_step2_tb", "k_step_fused", "k_step_fused_tma", "k_propagate", "k_propagate_tma", "k_collide", "k_bc",
       "k_pbc_wrap", "k_tb_pull", "k_peer_pull")


def demangle(names):
    try:
        r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
        return r.stdout.splitlines()
    except Exception:
        return names


def census(so: str = SO) -> dict:
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    funcs = {}
    cur = None
    for line in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            op = m.group(1)
            funcs[cur]["total"] += 1
            for k in OPS:
                if op == k:
                    funcs[cur][k] += 1
    mangled = list(funcs)
    out = {}
    for mg, dm in zip(mangled, demangle(mangled)):
        short = dm.replace("(anonymous namespace)::", "").replace("lbk::", "")
        short = re.sub(r"\(.*$", "", short)                    # drop the parameter list
        short = re.sub(r"^void ", "", short)
        base = re.sub(r"<.*$", "", short)
        c = funcs[mg]
        out[short] = {"kernel": base, **{k: c.get(k, 0) for k in ["total"] + OPS}}
    return out


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--so", default=SO)
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    res = census(a.so)
    hot = {k: v for k, v in res.items() if v["kernel"] in HOT}
    doc = {"what": "static SASS instruction counts per kernel of liblb_d2q37.so (cuobjdump -sass), sm_100a; "
                   "tools/sass_census.py",
           "hot_kernels_with_local_memory": [k for k, v in hot.items() if v["LDL"] or v["STL"]],
           "kernels": res}
    js = json.dumps(doc, indent=1)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(js + "\n")
    else:
        sys.stdout.write(js + "\n")
    return doc


if __name__ == "__main__":
    main()
