"""Where the e2e time goes (bench.py's e2e leg, 1920x2048): pinned H2D / D2H
bandwidth, lb_set_state, K steps with and without monitors, lb_gather.

usage (GPU box): python tools/e2e_breakdown.py [K]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import lbgen  # noqa: E402
from paper_1703_00186_b200 import lb  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
LX, LY = 1920, 2048
res = {}


def timed(name, fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    res[name] = round((time.perf_counter() - t) * 1e3, 3)


n = 37 * LX * LY
host = torch.empty(n, dtype=torch.float64).pin_memory()
dev = torch.empty(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    timed("raw_h2d_ms", lambda: dev.copy_(host, non_blocking=True))
    timed("raw_d2h_ms", lambda: host.copy_(dev, non_blocking=True))
res["raw_h2d_gbs"] = round(n * 8 / res["raw_h2d_ms"] / 1e6, 1)
res["raw_d2h_gbs"] = round(n * 8 / res["raw_d2h_ms"] / 1e6, 1)
del dev

g = lb.Lattice(LX, LY, tau=0.8, t_bottom=1.02, t_top=0.98, mode="fused")
if os.environ.get("TB_PDL") is not None:  # programmatic dependent launch on / off (default: library default)
    g.temporal(True, pdl=bool(int(os.environ["TB_PDL"])))
fields = lbgen.rt_macro(LX, LY, 1.0)
g.init_macro(*fields)
host.numpy()[:] = g.peek(0).reshape(-1)
out = torch.empty((37, LX, LY), dtype=torch.float64).pin_memory()
mon = torch.empty((K, 5), dtype=torch.float64).pin_memory()
for _ in range(2):
    timed("set_state_ms", lambda: g.set_state(host.numpy()))
    timed("steps_plain_ms", lambda: g.step(K))
    g.monitor(True)

    def mon_steps():
        for k in range(K):
            g.step(1)
            g.invariants_async(mon[k])
    timed("steps_monitored_ms", mon_steps)
    g.monitor(False)

    def loop_plain():
        for k in range(K):
            g.step(1)
    timed("steps_plain_loop_ms", loop_plain)
    g.monitor(True)

    def pair_steps():   # the two-step kernel with monitors of both states (bench e2e loop)
        for k in range(0, K, 2):
            g.step(2)
            g.invariants_pair_async(mon[k:k + 2])
    timed("steps_pair_monitored_ms", pair_steps)
    g.monitor(False)
    timed("gather_ms", lambda: g.gather(out=out.numpy()))
g.monitor(True)
g.profile(True)
g.profile_reset()
for k in range(200):
    g.step(1)
    g.invariants_async(mon[k])
g.sync()
res["profile_monitored_200"] = {k: round(v["total_ms"] / v["launches"] * 1e3, 2) for k, v in g.profile_read().items()
                                if v["launches"]}
g.profile_reset()
for k in range(0, 200, 2):
    g.step(2)
    g.invariants_pair_async(mon[k:k + 2])
g.sync()
res["profile_pair_monitored_200"] = {k: round(v["total_ms"] / v["launches"] * 1e3, 2)
                                     for k, v in g.profile_read().items() if v["launches"]}
g.profile(False)
g.monitor(False)
res["K"] = K
print(json.dumps(res))
