"""Small target for ncu: a few fused steps and a few split steps at 1920x2048.

ncu --set full -k regex:'k_step_fused|k_propagate|k_collide|k_bc' ... python tools/ncu_target.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402

lx, ly = int(os.environ.get("LB_LX", 1920)), int(os.environ.get("LB_LY", 2048))
fields = lbgen.rt_macro(lx, ly, lb.t0())
for mode in sys.argv[1:] or ["fused", "split"]:
    g = lb.Lattice(lx, ly, mode=mode)
    g.init_macro(*fields)
    g.step(3)
    g.sync()
    g.close()
    del g
    torch.cuda.empty_cache()
print("ncu target done")
