"""Fit the paper's §5 timing model to B200 kernel timings and
predict strong / weak scaling of BASELINE configs #3 / #4.

    python tools/timing_model.py [--out profiles/r01_timing_model.json]

alpha, beta: whole-lattice fused step kernel time over a grid of (Lx, Ly);
delta: border-column kernel time of the overlapped schedule (N = 1 run through
the NCCL 1-rank ring) over Ly; gamma: halo bytes per row (2 x 3 x 37 x 8 B,
both neighbours) over the NVLink peer-copy bandwidth measured on this pool
(770 GB/s per direction, B200_PROFILING.md) -- an input, not a measurement,
since the pool gives one GPU per job.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def kernel_ms(lb, lbgen, lx, ly, steps=20, **kw):
    g = lb.Lattice(lx, ly, temporal=False, **kw)  # the one-step kernel (the multi-GPU path)
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    g.step(3)
    g.profile(True)
    g.profile_reset()
    g.step(steps)
    prof = g.profile_read()
    g.close()
    return {k: v["total_ms"] / v["launches"] for k, v in prof.items() if v["launches"]}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--link-gbs", type=float, default=770.0)
    ap.add_argument("--eps-us", type=float, default=15.0, help="exchange latency for the extended model")
    a = ap.parse_args(argv)

    import torch

    import lbgen
    import paper_1703_00186_b200 as lb
    from paper_1703_00186_b200 import perfmodel as pm

    bulk = []
    for lx in (256, 512, 1024, 2048):
        for ly in (1024, 2048, 4096, 8192):
            t = kernel_ms(lb, lbgen, lx, ly)["k_step_fused"] * 1e-3
            bulk.append((lx, ly, t))
            torch.cuda.empty_cache()
    alpha, beta = pm.fit_bulk(bulk)
    border = []
    for ly in (1024, 2048, 4096, 8192):
        # a fresh NCCL unique id per communicator (an id bootstraps one init)
        t = kernel_ms(lb, lbgen, 64, ly, overlap=True, nccl_id=lb.nccl_unique_id())
        border.append((ly, t["k_step_fused_border"] * 1e-3))
    delta = pm.fit_rows(border)
    gamma = pm.exchange_gamma(2 * 3 * 37 * 8, a.link_gbs * 1e9)
    p = pm.Params(alpha, beta, gamma, delta)
    pe = pm.Params(alpha, beta, gamma, delta, eps=a.eps_us * 1e-6)
    pred = {}
    for name, (lx, ly, kind) in {"#3 strong 8192x8192": (8192, 8192, "strong"),
                                 "#4 weak 4096x8192/GPU": (4096, 8192, "weak"),
                                 "bench weak 1920x2048/GPU": (1920, 2048, "weak"),
                                 "paper 1080x5736 strong (P:809-820)": (1080, 5736, "strong")}.items():
        rows = []
        for n in (1, 2, 4, 8, 16, 24, 36, 48):
            if kind == "strong":
                rows.append({"n": n, "T_ms": pm.step_time(p, lx, ly, n) * 1e3, "S_r": pm.speedup(p, lx, ly, n),
                             "eff": pm.speedup(p, lx, ly, n) / n, "eff_with_eps": pm.speedup(pe, lx, ly, n) / n})
            else:
                rows.append({"n": n, "T_ms": pm.step_time(p, n * lx, ly, n) * 1e3,
                             "eff": pm.weak_efficiency(p, lx, ly, n),
                             "eff_with_eps": pm.weak_efficiency(pe, lx, ly, n)})
        pred[name] = rows
    res = {"params": p.as_dict(), "eps_s": pe.eps, "bulk_samples": bulk, "border_samples": border,
           "gamma_source": f"{2 * 3 * 37 * 8} B/row over {a.link_gbs} GB/s NVLink peer copy (B200_PROFILING.md)",
           "alpha_equiv_gbs": 592 / alpha / 1e9, "predictions": pred}
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    print(json.dumps({"params": res["params"], "alpha_equiv_gbs": res["alpha_equiv_gbs"],
                      "strong8192_eff": [round(r["eff"], 3) for r in pred["#3 strong 8192x8192"]][:4],
                      "weak4096_eff": [round(r["eff"], 3) for r in pred["#4 weak 4096x8192/GPU"]][:4]}))
    return res


if __name__ == "__main__":
    main()
