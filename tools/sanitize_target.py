"""Small target exercising every kernel of liblb_d2q37.so, for
compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402

lx, ly = 64, 32
T0 = lb.t0()
fields = lbgen.rt_macro(lx, ly, T0)
for bc in ("thermal", "adiabatic", "periodic"):
    for mode in ("fused", "split"):
        for coll in ("bgk", "regularized"):
            g = lb.Lattice(lx, ly, bc_y=bc, mode=mode, collision=coll, gravity=(0.0, -1e-5))
            g.init_macro(*fields)
            g.step(2)
            g.monitor(True)
            g.step(1)
            g.invariants()
            g.set_state(g.gather())
            g.exchange()
            g.peek(0)
            g.close()
# two-step kernel (temporal blocking): several strips incl. moved ones, both
# walls, monitors on and off, a small grid (several sweeps per CTA)
for (lx2, ly2), grid in (((40, 250), 0), ((24, 30), 0), ((17, 131), 3)):
    f2 = lbgen.rt_macro(lx2, ly2, T0)
    for coll in ("bgk", "regularized"):
        g = lb.Lattice(lx2, ly2, collision=coll, gravity=(1e-6, -1e-5))
        g.temporal(True, grid=grid)
        g.init_macro(*f2)
        g.step(2)
        g.monitor(True)
        g.step(2)
        buf = np.zeros(10)
        g.invariants_pair_async(buf)
        g.invariants()
        g.close()
# NCCL 1-rank ring with the overlapped schedule
g = lb.Lattice(lx, ly, overlap=True, nccl_id=lb.nccl_unique_id())
g.init_macro(*fields)
g.step(2)
g.invariants()
g.close()
# peer-store ring of 2 contexts on 2 streams
r = [lb.Lattice(lx * 2, ly, rank=k, nranks=2, stream=torch.cuda.Stream()) for k in range(2)]
for k, x in enumerate(r):
    x.init_macro(*lbgen.rt_macro(lx * 2, ly, T0, x0=k * lx, lx=lx))
r[0].set_peers(r[1], r[1])
r[1].set_peers(r[0], r[0])
torch.cuda.synchronize()
for _ in range(3):
    for x in r:
        x.step(1)
for x in r:
    x.sync()
# two-step kernel at N > 1: the in-kernel exchange (edge CTAs wait and read
# the neighbours' buffers by TMA, the last CTA signals) + two-step launches +
# a one-step remainder (waiting halo pull), monitors on; then the same with
# the staged exchange (k_tb_wait + k_tb_pull before the kernel, k_signal after)
for x in r:
    x.monitor(True)
for edge in (True, False):
    for x in r:
        x.edge_pull(edge)
    for _ in range(2):
        for x in r:
            x.step(2)
    for x in r:
        x.step(1)
    for x in r:
        x.sync()
print("sanitize target done", np.isfinite(r[0].peek(0)).all())
