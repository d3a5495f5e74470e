"""ncu target: a few launches of the two-step kernel at 1920x2048 (tools only)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lbm  # noqa: E402

lx, ly = 1920, 2048
coll = sys.argv[1] if len(sys.argv) > 1 else "bgk"
g = lbm.Lattice(lx, ly, collision=coll, temporal=True)
if os.environ.get("LB_TB_MON"):  # the monitored kernel (k_step2_tb<..., MON = true>)
    g.monitor(True)
if os.environ.get("LB_TB_PROMO"):
    g.temporal(True, l2_promotion=int(os.environ["LB_TB_PROMO"]))
g.init_macro(*lbgen.rt_macro(lx, ly, 1.0 / 1.19697977039307435897239 ** 2))
g.step(8)
g.sync()
torch.cuda.synchronize()
