"""The paper's §5 timing model refitted to the SHIPPED path: the
two-step kernel (two time steps per launch) with its N > 1 exchange either
serialised (k_tb_pull before the kernel) or inside the kernel (edge CTAs wait
and stage, the default).  Predicts N = 8 efficiencies of BASELINE configs #3
(strong, 8192x8192) and #4 (weak, 4096x8192 per GPU).  Measurement tool.

    python tools/timing_model_tb.py [--link-gbs 770] [--out profiles/r02_timing_model.json]

Per launch of 2 steps on n GPUs (slab lx = Lx/n):
    T_ser(n)  = alpha2 lx Ly + beta2 lx + [n > 1] (T_pull(Ly) + T_sig)
    T_ovl(n)  = alpha2 lx Ly + beta2 lx + [n > 1] T_edge(Ly)
alpha2, beta2: least squares over k_step2_tb launches at N = 1 (CUDA events);
T_pull: the k_tb_pull launch of an in-process ring on this GPU (its copy is
local here) or the NVLink time of its bytes, whichever is larger; T_edge:
the extra per-launch time of the in-kernel edge pull measured on the same
ring (shared stream, each launch alone on the GPU) plus the NVLink time of one
edge CTA's 6-column rows; T_sig: the k_signal launch (serialised path only:
the in-kernel exchange publishes its counter from the kernel's last CTA).  The pool has one GPU,
so the NVLink terms are inputs (B200_PROFILING.md's peer-copy rate), not
measurements.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402
from paper_1703_00186_b200 import perfmodel as pm  # noqa: E402

HT = lb.tb_strip_height()


def n1_launch_ms(lx, ly, pairs=20):
    g = lb.Lattice(lx, ly, stream=torch.cuda.Stream())
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    g.step(6)
    g.sync()
    g.profile(True)
    g.profile_reset()
    g.step(2 * pairs)
    p = g.profile_read()["k_step2_tb"]
    g.close()
    return p["total_ms"] / p["launches"]


def ring_ms(n, lx, ly, edge_pull, pairs=20):
    s = torch.cuda.Stream()
    T0 = lb.t0()
    ranks = [lb.Lattice(lx * n, ly, rank=r, nranks=n, stream=s) for r in range(n)]
    for r, g in enumerate(ranks):
        g.init_macro(*lbgen.rt_macro(lx * n, ly, T0, x0=r * lx, lx=lx))
        g.edge_pull(edge_pull)
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % n], ranks[(r + 1) % n])
    for _ in range(3):
        for g in ranks:
            g.step(2)
    for g in ranks:
        g.sync()
        g.profile(True)
        g.profile_reset()
    for _ in range(pairs):
        for g in ranks:
            g.step(2)
    out = {}
    for g in ranks:
        g.sync()
        for k, v in g.profile_read().items():
            out.setdefault(k, []).append(v["total_ms"] / v["launches"])
        g.close()
    torch.cuda.empty_cache()
    return {k: sum(v) / len(v) for k, v in out.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--link-gbs", type=float, default=770.0)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    link = a.link_gbs * 1e9
    bulk = []
    for lx in (256, 512, 1024, 2048):
        for ly in (1024, 2048, 4096, 8192):
            bulk.append((lx, ly, n1_launch_ms(lx, ly) * 1e-3))
            torch.cuda.empty_cache()
    alpha2, beta2 = pm.fit_bulk(bulk)
    ex = {}
    for ly in (2048, 4096, 8192):
        lx = 1024
        t1 = n1_launch_ms(lx, ly)
        ser = ring_ms(4, lx, ly, False)
        ovl = ring_ms(4, lx, ly, True)
        nyp = (16 + ly + 3 + 15) // 16 * 16
        pull_bytes = 2 * 6 * 37 * nyp * 8               # both sides, whole columns
        edge_bytes = 6 * 37 * (HT + 12) * 8             # one edge CTA, one side
        ex[ly] = {"n1_launch_ms": t1, "ring_k_step2_tb_ms_serialised": ser["k_step2_tb"],
                  "k_tb_pull_ms": ser["k_tb_pull"], "k_signal_ms": ser["k_signal"],
                  "ring_k_step2_tb_ms_in_kernel": ovl["k_step2_tb"],
                  "pull_nvlink_ms": pull_bytes / 2 / link * 1e3,    # two neighbours in parallel
                  "edge_nvlink_ms": edge_bytes / link * 1e3,
                  "T_pull_ms": max(ser["k_tb_pull"], pull_bytes / 2 / link * 1e3),
                  "T_edge_ms": max(0.0, ovl["k_step2_tb"] - t1) + edge_bytes / link * 1e3,
                  "T_sig_ms": ser["k_signal"]}
        print(ly, json.dumps(ex[ly]), flush=True)

    def terms(ly):
        # linear interpolation in ly of the measured exchange terms
        ks = sorted(ex)
        lo = max([k for k in ks if k <= ly] or [ks[0]])
        hi = min([k for k in ks if k >= ly] or [ks[-1]])
        f = 0.0 if hi == lo else (ly - lo) / (hi - lo)
        return {k: ex[lo][k] + f * (ex[hi][k] - ex[lo][k]) for k in ("T_pull_ms", "T_edge_ms", "T_sig_ms")}

    def t_launch(lx_slab, ly, n, mode):
        t = (alpha2 * lx_slab * ly + beta2 * lx_slab) * 1e3
        if n > 1:
            e = terms(ly)
            # serialised: k_tb_pull + kernel + k_signal; in-kernel: the edge
            # CTAs' waits and peer reads, and the kernel's last CTA signals
            t += e["T_pull_ms"] + e["T_sig_ms"] if mode == "serialised" else e["T_edge_ms"]
        return t

    pred = {}
    for name, (lx, ly, kind) in {"#3 strong 8192x8192": (8192, 8192, "strong"),
                                 "#4 weak 4096x8192/GPU": (4096, 8192, "weak"),
                                 "bench weak 1920x2048/GPU": (1920, 2048, "weak")}.items():
        rows = []
        for n in (1, 2, 4, 8):
            r = {"n": n}
            for mode in ("serialised", "overlapped"):
                if kind == "strong":
                    t1, tn = t_launch(lx, ly, 1, mode), t_launch(lx / n, ly, n, mode)
                    r[mode] = {"T_launch_ms": tn, "eff": t1 / (n * tn), "mlups": lx * ly * 2 / tn / 1e3}
                else:
                    t1, tn = t_launch(lx, ly, 1, mode), t_launch(lx, ly, n, mode)
                    r[mode] = {"T_launch_ms": tn, "eff": t1 / tn, "mlups": n * lx * ly * 2 / tn / 1e3}
            rows.append(r)
        pred[name] = rows
    res = {"what": __doc__.split("\n\n")[0], "alpha2_s_per_site_launch": alpha2, "beta2_s_per_column_launch": beta2,
           "alpha2_equiv_mlups": 2 / alpha2 / 1e6, "bulk_samples": bulk, "exchange_terms": ex,
           "link_gbs_input": a.link_gbs, "predictions": pred}
    js = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(js + "\n")
    print(json.dumps({name: [(r["n"], round(r["serialised"]["eff"], 4), round(r["overlapped"]["eff"], 4))
                             for r in rows] for name, rows in pred.items()}))


if __name__ == "__main__":
    main()
