"""BASELINE config #5: D2Q37 fp64 2048x4096 Rayleigh-Taylor long run (test infrastructure).

    python tests/long_run.py [--steps 10000] [--every 100] [--ckpt-every 1000]
                             [--check 10] [--gravity 0] [--nslabs 8] [--compare-n1]
                             [--out profiles/r02_long_run_n8.json]

The library runs `steps` steps of the lattice split into `nslabs` X-slabs
(BASELINE configs[4]: 8 slabs of 256 columns, the N = 8 geometry).  The pool
gives one GPU, so the slabs are an in-process ring on that GPU: one lattice
context per slab, exchanging only through the peer path (lb_set_peers: the two-step kernel's in-kernel edge pulls and step
counters) — the same code a one-GPU-per-rank run executes, with the peer
pointers local instead of CUDA-IPC mappings.  The slabs share one stream
(see Ring) so the ring cannot starve itself of SMs on a single GPU.  Every
`every` steps the
invariants (lb_invariants per slab, summed) record mass, momentum, energy and
the minimum density.  Every `ckpt-every` steps the state is saved as an
LBFIELD checkpoint and

* the library RESTARTS from the file (checkpoint.load + set_state per slab,
  the product's restart path) and continues from it;
* with --compare-n1, an unsplit (1-slab) lattice stepped alongside from
  memory must equal the file bit for bit (N == 1);
* the CPU oracle restarts from the same file, runs `check` steps, and must
  match the library's state `check` steps later within 1e-12 max relative
  error.
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


class Ring:
    """`n` X-slabs of one lattice in this process, exchanging through peer
    memory (n = 1: a plain single lattice, its own N = 1 wrap)."""

    def __init__(self, lb, lx_total, ly, n, **kw):
        import torch
        import lbgen
        self.n, self.lx_total, self.ly = n, lx_total, ly
        self.lx = lx_total // n
        self.slabs = []
        # ONE stream for all slabs: their launches run in issue order (slab
        # 0..n-1 for launch k, then k+1), so every counter wait is already
        # satisfied when a launch starts.  Separate streams would let up to n
        # kernels of 148 persistent CTAs, whose edge CTAs spin on counters,
        # compete for the SMs of this one GPU — a schedule a real
        # one-GPU-per-rank run never has (tests/test_gpu_parity.py covers
        # separate streams at grid sizes that stay co-resident).
        st = torch.cuda.Stream() if n > 1 else None
        for r in range(n):
            self.slabs.append(lb.Lattice(lx_total, ly, rank=r, nranks=n, stream=st, **kw))
        for r, g in enumerate(self.slabs):
            g.init_macro(*lbgen.rt_macro(lx_total, ly, lb.t0(), x0=r * self.lx, lx=self.lx))
        if n > 1:
            for r, g in enumerate(self.slabs):
                g.set_peers(self.slabs[(r - 1) % n], self.slabs[(r + 1) % n])
        torch.cuda.synchronize()

    def step(self, k):
        # interleave the slabs per launch (2 steps, or an odd remainder of 1):
        # on the one shared stream, slab r's launch j+1 waits for its
        # neighbours' launch j, which must already be queued ahead of it
        while k > 0:
            s = 2 if k >= 2 else 1
            for g in self.slabs:
                g.step(s)
            k -= s

    def sync(self):
        for g in self.slabs:
            g.sync()

    def state(self) -> np.ndarray:
        self.sync()
        return np.concatenate([g.peek(0) for g in self.slabs], axis=1)

    def set_state(self, full: np.ndarray):
        self.sync()
        for r, g in enumerate(self.slabs):
            g.set_state(np.ascontiguousarray(full[:, r * self.lx:(r + 1) * self.lx, :]))

    def invariants(self) -> np.ndarray:
        """[sum rho, sum jx, sum jy, sum E, min rho] over all slabs (the slabs'
        partial sums added in rank order)."""
        self.sync()
        inv = [g.invariants() for g in self.slabs]
        out = np.sum([v[:4] for v in inv], axis=0)
        return np.append(out, min(v[4] for v in inv))

    def launches(self):
        return sum(g.launch_count() for g in self.slabs)

    def close(self):
        for g in self.slabs:
            g.close()


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
    ap.add_argument("--nslabs", type=int, default=1, help="X-slabs of the in-process peer ring (8: configs[4])")
    ap.add_argument("--compare-n1", action="store_true", help="step an unsplit lattice alongside; bitwise checks")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)

    import oracle
    import paper_1703_00186_b200 as lb
    from paper_1703_00186_b200 import checkpoint

    grav = (0.0, -abs(a.gravity))
    coll_o = oracle.REGULARIZED if a.collision == "regularized" else oracle.BGK
    ring = Ring(lb, a.lx, a.ly, a.nslabs, collision=a.collision, gravity=grav)
    ref = Ring(lb, a.lx, a.ly, 1, collision=a.collision, gravity=grav) if (a.compare_n1 and a.nslabs > 1) else None
    inv0 = ring.invariants()
    series, checks, n1 = [], [], []
    tmp = tempfile.mkdtemp()
    t_gpu = 0.0
    step = 0
    launches0 = ring.launches()
    while step < a.steps:
        if step % a.ckpt_every == 0:
            path = os.path.join(tmp, f"ckpt_{step}.lbfield")
            checkpoint.save(path, ring.state())
            st = checkpoint.load(path)
            if ref is not None:
                n1.append({"step": step, "bitwise_equal_to_unsplit": bool(np.array_equal(st, ref.state()))})
            ring.set_state(st)          # the product's restart path: continue from the file
            ring.step(a.check)
            if ref is not None:
                ref.step(a.check)
            got = ring.state()
            o = oracle.Lattice(a.lx, a.ly, collision=coll_o, gravity=grav)
            o.set_state(st)
            t = time.perf_counter()
            o.step(a.check)
            t_or = time.perf_counter() - t
            want = o.get_state(0)
            err = float(np.max(np.abs(got - want) / np.abs(want)))
            checks.append({"step": step, "steps_checked": a.check, "max_rel_err": err,
                           "oracle_s": round(t_or, 2), "min_f": float(want.min())})
            os.remove(path)
            del o, st, got, want
            step += a.check
            continue
        k = min(a.every - step % a.every, a.steps - step, a.ckpt_every - step % a.ckpt_every)
        ring.sync()
        t = time.perf_counter()
        ring.step(k)
        ring.sync()
        t_gpu += time.perf_counter() - t
        if ref is not None:
            ref.step(k)
        step += k
        if step % a.every == 0:
            inv = ring.invariants()
            rec = {"step": step, "mass": inv[0], "jx": inv[1], "jy": inv[2], "energy": inv[3], "min_rho": inv[4]}
            if ref is not None:
                iv = ref.invariants()
                rec["unsplit_mass_rel_diff"] = float((inv[0] - iv[0]) / iv[0])
            series.append(rec)
    if ref is not None:
        n1.append({"step": step, "bitwise_equal_to_unsplit": bool(np.array_equal(ring.state(), ref.state()))})
    inv = ring.invariants()
    res = {
        "config": f"BASELINE #5: D2Q37 fp64 {a.lx}x{a.ly} RT, {a.steps} steps, thermal walls, tau 0.8, "
                  f"g = {grav}, collision {a.collision}, {a.nslabs} X-slab(s) of {a.lx // a.nslabs} columns"
                  + (" as an in-process peer ring on one GPU" if a.nslabs > 1 else ""),
        "nslabs": a.nslabs, "steps": a.steps, "mass0": inv0[0], "mass_final": inv[0],
        "rel_mass_drift": (inv[0] - inv0[0]) / inv0[0],
        "min_rho_final": inv[4],
        "gpu_mlups_between_checks": a.lx * a.ly * (a.steps - len(checks) * a.check) / t_gpu / 1e6
        if t_gpu > 0 else None,
        "kernel_launches": ring.launches() - launches0,
        "restart_from_file": True,
        "checkpoint_restart_parity": checks,
        "max_checkpoint_err": max(c["max_rel_err"] for c in checks) if checks else None,
        "unsplit_bitwise": n1,
        "all_bitwise_equal_to_unsplit": all(c["bitwise_equal_to_unsplit"] for c in n1) if n1 else None,
        "invariants_every": a.every, "series": series,
    }
    ring.close()
    if ref is not None:
        ref.close()
    if a.out:
        with open(a.out, "w") as fh:
            json.dump(res, fh, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "series"}))
    return res


if __name__ == "__main__":
    main()
