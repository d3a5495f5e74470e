"""BASELINE config #5 on one GPU: D2Q37 fp64 2048x4096 Rayleigh-Taylor long run.

    python tests/long_run.py [--steps 10000] [--every 100] [--ckpt-every 1000]
                             [--check 10] [--gravity 0] [--out profiles/r01_long_run.json]

The fused GPU path runs `steps` steps; lb_invariants every `every` steps
records total mass, momentum, energy and the minimum site density.  At every
`ckpt-every` steps the state is gathered and saved as an LBFIELD checkpoint;
the CPU oracle restarts from it, runs `check` steps, and must match the GPU's
state `check` steps later within 1e-12 max relative error.
The N=8 version of the run is the same code under torchrun; this pool gives
one GPU, so the lattice runs unsplit.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--lx", type=int, default=2048)
    ap.add_argument("--ly", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10000)
    ap.add_argument("--every", type=int, default=100)
    ap.add_argument("--ckpt-every", type=int, default=1000)
    ap.add_argument("--check", type=int, default=10)
    ap.add_argument("--gravity", type=float, default=0.0, help="g_y < 0 pulls down (RT dynamics)")
    ap.add_argument("--collision", default="bgk")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)

    import lbgen
    import oracle
    import paper_1703_00186_b200 as lb
    from paper_1703_00186_b200 import checkpoint

    grav = (0.0, -abs(a.gravity))
    coll_o = oracle.REGULARIZED if a.collision == "regularized" else oracle.BGK
    g = lb.Lattice(a.lx, a.ly, collision=a.collision, gravity=grav)
    g.init_macro(*lbgen.rt_macro(a.lx, a.ly, lb.t0()))
    inv0 = g.invariants()
    series, checks = [], []
    tmp = tempfile.mkdtemp()
    t_gpu = 0.0
    step = 0
    while step < a.steps:
        if step % a.ckpt_every == 0:
            st = g.gather()
            path = os.path.join(tmp, f"ckpt_{step}.lbfield")
            checkpoint.save(path, st)
            g.step(a.check)
            got = g.gather()
            o = oracle.Lattice(a.lx, a.ly, collision=coll_o, gravity=grav)
            o.set_state(checkpoint.load(path))
            t = time.perf_counter()
            o.step(a.check)
            t_or = time.perf_counter() - t
            ref = o.get_state(0)
            err = float(np.max(np.abs(got - ref) / np.abs(ref)))
            checks.append({"step": step, "steps_checked": a.check, "max_rel_err": err,
                           "oracle_s": round(t_or, 2), "min_f": float(ref.min())})
            os.remove(path)
            del o, st, got, ref
            step += a.check
            continue
        n = min(a.every - step % a.every, a.steps - step, a.ckpt_every - step % a.ckpt_every)
        g.sync()
        t = time.perf_counter()
        g.step(n)
        g.sync()
        t_gpu += time.perf_counter() - t
        step += n
        if step % a.every == 0:
            inv = g.invariants()
            series.append({"step": step, "mass": inv[0], "jx": inv[1], "jy": inv[2], "energy": inv[3],
                           "min_rho": inv[4]})
    inv = g.invariants()
    res = {
        "config": f"BASELINE #5 on 1 GPU: D2Q37 fp64 {a.lx}x{a.ly} RT, {a.steps} steps, thermal walls, "
                  f"tau 0.8, g = {grav}, collision {a.collision}",
        "steps": a.steps, "mass0": inv0[0], "mass_final": inv[0],
        "rel_mass_drift": (inv[0] - inv0[0]) / inv0[0],
        "min_rho_final": inv[4], "gpu_mlups_between_checks": a.lx * a.ly * (a.steps - len(checks) * a.check) / t_gpu / 1e6
        if t_gpu > 0 else None,
        "checkpoint_restart_parity": checks,
        "max_checkpoint_err": max(c["max_rel_err"] for c in checks) if checks else None,
        "invariants_every": a.every, "series": series,
    }
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "series"}))
    return res


if __name__ == "__main__":
    main()
