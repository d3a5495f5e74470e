"""Per-CTA timeline of one two-step launch (tools only).

LB_D2Q37_LIB=paper_1703_00186_b200/variants/liblb_<tag>.so [TB_WW=w16] python tools/tb_clock.py [lx ly] [out.json]

The variant must be built with LB_TB_CLOCK=1 (tools/build_tb_variant.py 104 1 1
LB_TB_CLOCK=1): every CTA of k_step2_tb records %globaltimer at its start and
end, its SM id, its sweep count and its iteration count.  Prints the spread of
CTA durations (max / mean: the tail the launch pays) and the slowest CTAs.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lbm  # noqa: E402


def main():
    lx, ly = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1920, 2048)
    out = sys.argv[3] if len(sys.argv) > 3 else None
    L = lbm.lib()
    fn = L.lb_debug_tb_clock
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
    res = {"lx": lx, "ly": ly, "launches": []}
    for coll in ("bgk", "regularized"):
        g = lbm.Lattice(lx, ly, collision=coll, temporal=True, bc_y=os.environ.get("TB_BC", "thermal"))
        if os.environ.get("TB_WW") or os.environ.get("TB_TW"):  # wall-strip / tail weights x16 (work split)
            g.temporal(True, wall_weight16=int(os.environ.get("TB_WW", "0")),
                       tail_weight16=int(os.environ.get("TB_TW", "0")))
        g.init_macro(*lbgen.rt_macro(lx, ly, 1.0 / 1.19697977039307435897239 ** 2))
        g.step(40)
        g.sync()
        for rep in range(3):
            g.step(2)
            g.sync()
            torch.cuda.synchronize()
            buf = np.zeros(4 * 1024, dtype=np.uint64)
            assert fn(buf.ctypes.data, 1024) == 0
            a = buf.reshape(1024, 4)
            G = int(np.count_nonzero(a[:, 1]))
            a = a[:G]
            t0 = a[:, 0].astype(np.int64)
            t1 = a[:, 1].astype(np.int64)
            dur = (t1 - t0) / 1e3
            start = (t0 - t0.min()) / 1e3
            end = (t1 - t0.min()) / 1e3
            sweeps = (a[:, 3] >> np.uint64(32)).astype(int)
            iters = (a[:, 3] & np.uint64(0xFFFFFFFF)).astype(int)
            rec = {"coll": coll, "rep": rep, "ctas": G, "launch_us": float(end.max()),
                   "dur_mean_us": float(dur.mean()), "dur_max_us": float(dur.max()), "dur_min_us": float(dur.min()),
                   "max_over_mean": float(dur.max() / dur.mean()), "start_max_us": float(start.max()),
                   "us_per_iter_mean": float((dur / iters).mean()),
                   "us_per_iter_min": float((dur / iters).min()), "us_per_iter_max": float((dur / iters).max()),
                   "iters_min": int(iters.min()), "iters_max": int(iters.max()),
                   "two_sweep_ctas": int((sweeps > 1).sum())}
            order = np.argsort(-dur)[:8]
            rec["slowest"] = [{"cta": int(i), "sm": int(a[i, 2]), "us": round(float(dur[i]), 2),
                               "iters": int(iters[i]), "sweeps": int(sweeps[i]),
                               "us_per_iter": round(float(dur[i] / iters[i]), 4)} for i in order]
            rec["per_cta"] = [[int(a[i, 2]), round(float(start[i]), 2), round(float(dur[i]), 2), int(iters[i]),
                               int(sweeps[i])] for i in range(G)]
            res["launches"].append(rec)
            print(json.dumps({k: v for k, v in rec.items() if k != "per_cta"}), flush=True)
        g.close()
    if out:
        with open(out, "w") as fh:
            json.dump(res, fh)


if __name__ == "__main__":
    main()
