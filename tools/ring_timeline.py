"""Per-launch cost of the N > 1 exchange of the two-step kernel (measurement tool).

    python tools/ring_timeline.py [--n 4] [--lx 1920] [--ly 2048] [--pairs 50]
                                  [--out profiles/r02_ring_timeline.json]

An in-process ring of N X-slabs of lx x ly each on ONE GPU (peer mode, the
same code a one-GPU-per-rank run executes).  Two schedules:

* shared stream: the slabs' launches are serialised on one stream (rank 0..N-1
  for pair k, then pair k+1), so every launch runs alone on the GPU and its
  CUDA-event duration is comparable with the N = 1 launch of the same slab
  size (periodic wrap, no exchange).  Compared: in-kernel edge pulls
  (LB_OPT_TB_EDGE_PULL = 1, default) vs k_tb_pull + kernel (0).
* separate streams (one per slab, as ranks would be): an event timeline of
  every launch (start / end on its stream, relative to one origin), showing
  the launches and the counter waits interleave without a host round trip.

Every configuration's final state is compared bit for bit with the unsplit
lattice stepped on the one-step kernel.
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lb  # noqa: E402


def make_ring(n, lx, ly, streams, edge_pull):
    T0 = lb.t0()
    ranks = [lb.Lattice(lx * n, ly, rank=r, nranks=n, stream=streams[r]) for r in range(n)]
    for r, g in enumerate(ranks):
        g.init_macro(*lbgen.rt_macro(lx * n, ly, T0, x0=r * lx, lx=lx))
        g.edge_pull(edge_pull)
    for r, g in enumerate(ranks):
        g.set_peers(ranks[(r - 1) % n], ranks[(r + 1) % n])
    torch.cuda.synchronize()
    return ranks


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--lx", type=int, default=1920)
    ap.add_argument("--ly", type=int, default=2048)
    ap.add_argument("--pairs", type=int, default=50)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    n, lx, ly, P = a.n, a.lx, a.ly, a.pairs
    res = {"what": f"in-process ring of {n} slabs of {lx}x{ly} on one B200 (peer mode, two-step kernel), "
                   f"{P} launches (= {2 * P} steps) per configuration after 3 warm-up launches; tools/ring_timeline.py"}

    # N = 1 reference launch time (periodic wrap, same slab size)
    s = torch.cuda.Stream()
    g = lb.Lattice(lx, ly, stream=s)
    g.init_macro(*lbgen.rt_macro(lx, ly, lb.t0()))
    g.step(6)
    g.sync()
    g.profile(True)
    g.profile_reset()
    g.step(2 * P)
    p = g.profile_read()["k_step2_tb"]
    n1 = p["total_ms"] / p["launches"]
    res["n1_launch_ms"] = n1
    g.close()

    # unsplit reference state (one-step kernel)
    ref = lb.Lattice(lx * n, ly, temporal=False)
    ref.init_macro(*lbgen.rt_macro(lx * n, ly, lb.t0()))
    ref.step(2 * (P + 3))
    want = ref.gather()
    ref.close()
    del ref
    torch.cuda.empty_cache()

    # shared stream: each launch alone on the GPU
    for edge_pull in (True, False):
        s = torch.cuda.Stream()
        ranks = make_ring(n, lx, ly, [s] * n, edge_pull)
        for _ in range(3):
            for g in ranks:
                g.step(2)
        for g in ranks:
            g.sync()
            g.profile(True)
            g.profile_reset()
        for _ in range(P):
            for g in ranks:
                g.step(2)
        for g in ranks:
            g.sync()
        per_rank = []
        for g in ranks:
            pr = g.profile_read()
            kt = pr["k_step2_tb"]
            d = {"k_step2_tb_ms": kt["total_ms"] / kt["launches"]}
            if "k_tb_pull" in pr:
                d["k_tb_pull_ms"] = pr["k_tb_pull"]["total_ms"] / pr["k_tb_pull"]["launches"]
            # (the in-kernel exchange publishes from the kernel: no k_signal)
            d["k_signal_ms"] = pr["k_signal"]["total_ms"] / pr["k_signal"]["launches"] if "k_signal" in pr else 0.0
            d["launch_sum_ms"] = d["k_step2_tb_ms"] + d.get("k_tb_pull_ms", 0.0) + d["k_signal_ms"]
            per_rank.append(d)
        got = np.concatenate([g.peek(0) for g in ranks], axis=1)
        key = "shared_stream_" + ("in_kernel_edge_pull" if edge_pull else "k_tb_pull")
        mean_sum = statistics.mean(d["launch_sum_ms"] for d in per_rank)
        res[key] = {"per_rank": per_rank, "mean_launch_sum_ms": mean_sum,
                    "vs_n1": mean_sum / n1, "bitwise_equal_to_unsplit": bool(np.array_equal(got, want))}
        for g in ranks:
            g.close()
        del ranks
        torch.cuda.empty_cache()
        print(key, json.dumps(res[key]), flush=True)

    # separate streams: event timeline.  Each slab's kernel gets 148 / n CTAs,
    # so all n kernels can be co-resident on this one GPU (with 148 CTAs each,
    # edge CTAs spinning on counters could starve the kernels they wait for —
    # a schedule a one-GPU-per-rank run never has)
    streams = [torch.cuda.Stream() for _ in range(n)]
    ranks = make_ring(n, lx, ly, streams, True)
    for g in ranks:
        g.temporal(True, grid=148 // n)
    for _ in range(3):
        for g in ranks:
            g.step(2)
    torch.cuda.synchronize()
    origin = torch.cuda.Event(enable_timing=True)
    origin.record(streams[0])
    for st in streams[1:]:
        st.wait_event(origin)
    ev = []
    T = min(P, 10)
    for k in range(T):
        for r, g in enumerate(ranks):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(streams[r])
            g.step(2)
            e1.record(streams[r])
            ev.append((r, k, e0, e1))
    for g in ranks:
        g.sync()
    torch.cuda.synchronize()
    tl = [{"rank": r, "launch": k, "start_ms": origin.elapsed_time(e0), "end_ms": origin.elapsed_time(e1)}
          for r, k, e0, e1 in ev]
    got = np.concatenate([g.peek(0) for g in ranks], axis=1)
    ref = lb.Lattice(lx * n, ly, temporal=False)
    ref.init_macro(*lbgen.rt_macro(lx * n, ly, lb.t0()))
    ref.step(2 * (T + 3))
    span = max(t["end_ms"] for t in tl) - min(t["start_ms"] for t in tl)
    res["separate_streams_timeline"] = {"grid_per_slab": 148 // n, "launches": tl, "span_ms": span,
                                        "span_per_launch_ms": span / (T * n),
                                        "bitwise_equal_to_unsplit": bool(np.array_equal(got, ref.gather()))}
    print("separate streams span/launch", span / (T * n), flush=True)
    js = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(js + "\n")
    print(json.dumps({k: v for k, v in res.items() if k != "separate_streams_timeline"}))


if __name__ == "__main__":
    main()
