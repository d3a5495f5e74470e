"""Small-lattice step rate with and without CUDA-graph stepping (config #1 size)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402

for lx, ly in ((64, 32), (256, 256), (1920, 2048)):
    res = {}
    for graphs in (False, True):
        st = torch.cuda.Stream()
        g = lb.Lattice(lx, ly, stream=st)
        if graphs:
            g.use_graphs(True)
        g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
        n = 2000 if lx * ly < 1e6 else 200
        g.step(20)
        g.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g.step(n)
        e1.record(st)
        g.sync()
        ms = e0.elapsed_time(e1) / n
        res["graph" if graphs else "plain"] = (round(ms * 1e3, 2), round(lx * ly / ms / 1e3, 1))
        g.close()
    print(f"{lx}x{ly}: us/step, MLUPS = {res}")
