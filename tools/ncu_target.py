"""Small target for ncu: a few steps per spec at 1920x2048.

spec = mode[:collision[:impl]]   e.g.  fused  split  fused:regularized  split:bgk:ldg  fused:bgk:tma  fused:bgk:tb
(fused specs without impl "tb" run the one-step kernel; "tb" the two-step kernel)
ncu ... python tools/ncu_target.py fused split fused:regularized split:regularized split:bgk:ldg
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402

lx, ly = int(os.environ.get("LB_LX", 1920)), int(os.environ.get("LB_LY", 2048))
fields = lbgen.rt_macro(lx, ly, lb.t0())
for spec in sys.argv[1:] or ["fused", "split"]:
    parts = spec.split(":")
    mode = parts[0]
    coll = parts[1] if len(parts) > 1 else "bgk"
    impl = parts[2] if len(parts) > 2 else None
    g = lb.Lattice(lx, ly, mode=mode, collision=coll, temporal=(impl == "tb"))
    if impl and impl != "tb":
        (g.set_propagate_impl if mode == "split" else g.set_fused_impl)(impl)
    g.init_macro(*fields)
    g.step(4 if impl == "tb" else 3)
    g.sync()
    g.close()
    del g
    torch.cuda.empty_cache()
print("ncu target done")
