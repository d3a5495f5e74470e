"""Where the config #5 mass drift comes from (measurement / analysis tool).

    python tools/drift_study.py [--lx 256] [--ly 4096] [--steps 1000] [--every 100]
                                [--side oracle|gpu|both] [--out profiles/r02_drift_study.json]

Per-step relative mass drift (least-squares slope of (M(n) - M(0)) / M(0)
over n, M every `every` steps summed over the whole state in long double —
the library's and the oracle's own invariants carry a summation error of
their own (the oracle's sequential sum over 10^7-10^8 values is ~1e-12
relative), larger than the drift being measured) of the RT workload under three wall
treatments — thermal walls (mirror + repopulation with K_wall), adiabatic
walls (mirror only: no K_wall), periodic Y (no walls at all) — on the CPU
oracle and/or the library, plus the exact (long double) rounding defect of
sum_l K_wall,l for both wall temperatures, which bounds the wall term.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import lbgen  # noqa: E402


def mass(state):
    """sum of every population of every site, accumulated in long double"""
    return float(np.sum(state, dtype=np.longdouble))


def slope(series):
    n = np.array([s[0] for s in series], dtype=float)
    m = np.array([s[1] for s in series], dtype=float)
    rel = (m - m[0]) / m[0]
    A = np.vstack([n - n[0], np.ones_like(n)]).T
    k, c = np.linalg.lstsq(A, rel, rcond=None)[0]
    resid = rel - (k * (n - n[0]) + c)
    return float(k), float(rel[-1]), float(np.abs(resid).max())


def run_oracle(lx, ly, steps, every, bc):
    import oracle
    o = oracle.Lattice(lx, ly, bc_y=bc)
    o.init_macro(*lbgen.rt_macro(lx, ly, oracle.t0()))
    series = [(0, mass(o.get_state(0)))]
    t = time.perf_counter()
    for n in range(every, steps + 1, every):
        o.step(every)
        series.append((n, mass(o.get_state(0))))
    return series, time.perf_counter() - t


def run_gpu(lx, ly, steps, every, bc):
    import paper_1703_00186_b200 as lb
    g = lb.Lattice(lx, ly, bc_y=bc)
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    series = [(0, mass(g.gather()))]
    for n in range(every, steps + 1, every):
        g.step(every)
        series.append((n, mass(g.gather())))
    g.close()
    return series


def kwall_defect():
    """sum_l K_wall,l - 1 in the doubles both sides use (oracle's K), evaluated
    exactly in long double, for T_bottom = 1.05 T0 and T_top = 0.95 T0."""
    import oracle
    out = {}
    for name, tw in (("bottom", 1.05 * oracle.t0()), ("top", 0.95 * oracle.t0())):
        K = oracle.kwall(tw).astype(np.longdouble)
        out[name] = float(K.sum() - np.longdouble(1.0))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lx", type=int, default=256)
    ap.add_argument("--ly", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--every", type=int, default=100)
    ap.add_argument("--side", default="oracle", choices=["oracle", "gpu", "both"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {"workload": f"RT init, {a.lx}x{a.ly}, tau 0.8, T_bottom 1.05 T0, T_top 0.95 T0, {a.steps} steps, "
                       f"mass every {a.every}",
           "sum_kwall_minus_1": kwall_defect()}
    bcs = {"thermal": 0, "adiabatic": 1, "periodic": 2}
    for side in (["oracle", "gpu"] if a.side == "both" else [a.side]):
        res[side] = {}
        for name, bc in bcs.items():
            if side == "oracle":
                series, secs = run_oracle(a.lx, a.ly, a.steps, a.every, bc)
            else:
                series, secs = run_gpu(a.lx, a.ly, a.steps, a.every, name), None
            k, last, dev = slope(series)
            res[side][name] = {"per_step_rel_drift": k, "rel_drift_at_end": last, "max_dev_from_line": dev,
                               "seconds": secs, "series": series}
            print(side, name, k, last, dev, flush=True)
    # the wall term's size if every band site's repopulation carried sum K - 1
    d = res["sum_kwall_minus_1"]
    res["wall_term_bound_per_step"] = 3 * (abs(d["bottom"]) + abs(d["top"])) / a.ly
    js = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(js + "\n")
    print(json.dumps({k: v for k, v in res.items() if k not in ("oracle", "gpu")}))


if __name__ == "__main__":
    main()
