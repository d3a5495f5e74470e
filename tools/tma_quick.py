import sys; sys.path.insert(0, '.')
import numpy as np, lbgen, oracle, paper_1703_00186_b200 as lb
lx, ly = 64, 32
st = lbgen.random_field(37, lx, ly, seed=3)
res = {}
for impl in ("ldg", "tma"):
    g = lb.Lattice(lx, ly, mode="split")
    if impl == "tma":
        g.set_propagate_impl("tma")
    g.set_state(st)
    outs = []
    for k in range(2):
        g.exchange(); g.propagate(); g.sync()
        outs.append(g.peek(1))
        g.bc(); g.collide()
    res[impl] = outs
for k in range(2):
    a, b = res["ldg"][k], res["tma"][k]
    d = np.argwhere(a != b)
    print("round", k, "ndiff", len(d), d[:10].tolist())
