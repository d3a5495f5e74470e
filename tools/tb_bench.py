"""Sweep of the two-step (temporal-blocking) kernel against the fused step.

python tools/tb_bench.py [lx ly] — MLUPS of lb_step(K) at 1920x2048 (default)
with LB_OPT_TEMPORAL off / on over a few CTA counts and L2 prefetch distances.
CUDA events on the context stream, warm-up first; device-resident inputs
(2 x 1.19 GB, far above L2).  Exploration tool, not the bench contract.
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__file__)))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lbm  # noqa: E402


def run(lx, ly, tb, grid=0, l2=0, k=None, coll="bgk", ww=0, promo=None, tw=0):
    k = k or int(os.environ.get("TB_K", "200"))
    s = torch.cuda.Stream()
    g = lbm.Lattice(lx, ly, collision=coll, stream=s, temporal=False)
    if tb:
        pdl = os.environ.get("TB_PDL")  # programmatic dependent launch on / off (unset: library default)
        g.temporal(True, grid=grid, l2_prefetch=l2, wall_weight16=ww, l2_promotion=promo, tail_weight16=tw,
                   pdl=None if pdl is None else bool(int(pdl)))
    g.init_macro(*lbgen.rt_macro(lx, ly, 1.0 / 1.19697977039307435897239 ** 2))
    g.step(20)
    g.sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.step(k)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / k
    out = g.gather()
    g.close()
    return ms, lx * ly / ms / 1e3, out


def main():
    lx, ly = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (1920, 2048)
    res = []
    ms, ml, ref = run(lx, ly, False)
    res.append({"tb": 0, "ms_per_step": ms, "mlups": ml})
    print(json.dumps(res[-1]), flush=True)
    grids = [int(x) for x in os.environ.get("TB_GRIDS", "0,296").split(",") if x]
    l2s = [int(x) for x in os.environ.get("TB_L2", "0,2,4,8").split(",") if x]
    for grid in grids:
        for l2 in l2s:
            ms, ml, out = run(lx, ly, True, grid, l2)
            res.append({"tb": 1, "grid": grid, "l2": l2, "ms_per_step": ms, "mlups": ml,
                        "bit_identical": bool(np.array_equal(out, ref))})
            print(json.dumps(res[-1]), flush=True)
    for ww in [int(x) for x in os.environ.get("TB_WW", "").split(",") if x]:
        ms, ml, out = run(lx, ly, True, 0, 0, ww=ww)
        print(json.dumps({"tb": 1, "wall_w16": ww, "ms_per_step": ms, "mlups": ml,
                          "bit_identical": bool(np.array_equal(out, ref))}), flush=True)
    for combo in [x for x in os.environ.get("TB_COMBOS", "").split(",") if x]:
        grid, ww = (int(v) for v in combo.split(":"))
        ms, ml, out = run(lx, ly, True, grid, 0, ww=ww)
        print(json.dumps({"tb": 1, "grid": grid, "wall_w16": ww, "ms_per_step": ms, "mlups": ml,
                          "bit_identical": bool(np.array_equal(out, ref))}), flush=True)
    wt_coll = os.environ.get("TB_WT_COLL", "bgk")
    if wt_coll != "bgk" and os.environ.get("TB_WT"):
        _, _, ref = run(lx, ly, False, coll=wt_coll)
    for combo in [x for x in os.environ.get("TB_WT", "").split(",") if x]:  # wall:tail weights x16
        ww, tw = (int(v) for v in combo.split(":"))
        ms, ml, out = run(lx, ly, True, 0, 0, ww=ww, tw=tw, coll=wt_coll)
        print(json.dumps({"tb": 1, "coll": wt_coll, "wall_w16": ww, "tail_w16": tw, "ms_per_step": ms, "mlups": ml,
                          "bit_identical": bool(np.array_equal(out, ref))}), flush=True)
    promos = [int(x) for x in os.environ.get("TB_PROMO", "").split(",") if x]
    if promos:
        _, _, ref_c = run(lx, ly, False, coll="regularized")
    for promo in promos:
        for coll in ("bgk", "regularized"):
            ms, ml, out = run(lx, ly, True, 0, 0, coll=coll, promo=promo)
            print(json.dumps({"tb": 1, "l2_promotion": promo, "coll": coll, "ms_per_step": ms, "mlups": ml,
                              "bit_identical": bool(np.array_equal(out, ref if coll == "bgk" else ref_c))}),
                  flush=True)
    for coll in ("regularized",):
        ms, ml, ref = run(lx, ly, False, coll=coll)
        print(json.dumps({"tb": 0, "coll": coll, "mlups": ml}), flush=True)
        ms, ml, out = run(lx, ly, True, coll=coll)
        print(json.dumps({"tb": 1, "coll": coll, "mlups": ml, "bit_identical": bool(np.array_equal(out, ref))}),
              flush=True)


if __name__ == "__main__":
    main()
