#!/usr/bin/env python
"""Benchmark of the D2Q37 hot path (BASELINE.json metric) — prints ONE JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config weak1920|strong8192|weak4096] [--mode fused|split]

A "step" is one full D2Q37 time step (pbc -> propagate -> bc -> collide, fused
pull kernel) over the whole lattice.  N = 1: config #2 of BASELINE.json, the
1920x2048 lattice; N > 1 (torchrun, one rank per GPU; halo exchange by peer
stores fused into the step kernel over CUDA-IPC/NVLink, or --transport nccl):
weak scaling with 1920x2048 per GPU (global lattice 1920N x 2048).  value =
lattice sites of all ranks x K / max-over-ranks device time (MLUPS).

Extra keys: roofline (dominant kernel k_step_fused vs the
measured HBM copy bandwidth), kernels (split-mode propagate / bc / collide per
kernel, collide FP64 % of the measured peak), e2e (same metric through the C
ABI with pinned host buffers: state upload, per-step invariants read-back,
final gather), clocks (NVML samples during the timed region), cpu_baseline
(the CPU oracle on a bounded sample of the same workload, rank 0 at N=1).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "D2Q37 fp64 MLUPS at 1/2/4/8 B200; propagate HBM GB/s, collide FP64 % of peak"
BYTES_PER_SITE = 592  # 37 fp64 reads + 37 fp64 writes (Table 1 convention)
CONFIGS = {
    # name: (lx per GPU or global, ly, scaling)
    "weak1920": (1920, 2048, "weak"),     # BASELINE configs[1] per GPU
    "weak4096": (4096, 8192, "weak"),     # BASELINE configs[3]
    "strong8192": (8192, 8192, "strong"), # BASELINE configs[2]
}


def load_json(path, default=None):
    try:
        with open(path) as fh:
            return json.load(fh)
    except Exception:
        return default


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.0002):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period = period
        self._stop = threading.Event()
        self._active = threading.Event()   # samples count only between begin() and end()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            if not self._active.is_set():
                self._active.wait(0.01)
                continue
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)   # ~0.4 ms per query
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                if self._active.is_set():
                    self.samples.append(mhz)
                    for bit, name in self.REASONS.items():
                        if r & bit and bit != 0x1:
                            self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def begin(self):
        self._active.set()

    def end(self):
        self._active.clear()

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._active.clear()
        self._stop.set()
        if self._t is not None:
            self._t.join()
            # one sample after the region too, in case it was shorter than the period
            if not self.samples:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))

    def summary(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ----------------------------------------------------------------------------- oracle leg

def oracle_throughput(lx_total: int, ly: int, budget_s: float):
    """The CPU oracle, as it stands, on a bounded sample of the workload: full
    time steps of the same RT lattice (the whole lattice if one step fits the
    budget, else its first w columns with all ly rows), as many steps as fit
    in about budget_s.  Returns (MLUPS, cores, sample description)."""
    import lbgen
    import oracle
    T0 = oracle.t0()
    probe_w = min(lx_total, 32)
    o = oracle.Lattice(probe_w, ly)
    o.init_macro(*lbgen.rt_macro(lx_total, ly, T0, lx=probe_w))
    o.step(1)
    t = time.perf_counter()
    o.step(1)
    per_site = (time.perf_counter() - t) / (probe_w * ly)
    w = int(max(3, min(lx_total, budget_s / (per_site * ly))))
    nsteps = int(max(1, min(1000, budget_s / (per_site * w * ly))))
    o = oracle.Lattice(w, ly)
    o.init_macro(*lbgen.rt_macro(lx_total, ly, T0, lx=w))
    t = time.perf_counter()
    o.step(nsteps)
    dt = time.perf_counter() - t
    mlups = w * ly * nsteps / dt / 1e6
    sample = (f"oracle lbref (C, -O2 -ffp-contract=off, OpenMP over ix) {nsteps} full step(s) on "
              f"columns 0..{w - 1} (all {ly} rows) of the {lx_total}x{ly} RT workload, {dt:.1f} s")
    return mlups, oracle.threads(), sample, dt, w, nsteps


def oracle_protocol():
    """SURVEY §8d oracle timing protocol: the oracle as it stands on 64x32 x 10
    steps and 1920x2048 x 3 steps (whole lattices, RT init), once with one
    thread and once with OpenMP over ix on all the host cores it may use.
    Returns {workload: {"threads_1": MLUPS, "threads_<n>": MLUPS, ...}}."""
    import lbgen
    import oracle
    T0 = oracle.t0()
    ncores = len(os.sched_getaffinity(0))
    res = {"cores_available": ncores}
    for lx, ly, nsteps in ((64, 32, 10), (1920, 2048, 3)):
        key = f"{lx}x{ly}_{nsteps}steps"
        res[key] = {}
        for nt in (1, ncores):
            oracle.set_threads(nt)
            o = oracle.Lattice(lx, ly)
            o.init_macro(*lbgen.rt_macro(lx, ly, T0))
            t = time.perf_counter()
            o.step(nsteps)
            dt = time.perf_counter() - t
            res[key][f"threads_{oracle.threads()}"] = round(lx * ly * nsteps / dt / 1e6, 3)
            del o
    oracle.set_threads(ncores)
    return res


def run_reference(args, cfg_name, lx_total, ly, scaling, rank, world):
    if rank != 0:
        return
    budget = float(os.environ.get("LB_REF_BUDGET_S", "60"))
    per_step = budget / max(1, args.steps + args.warmup)
    import oracle
    import lbgen
    T0 = oracle.t0()
    probe_w = min(lx_total, 16)
    o = oracle.Lattice(probe_w, ly)
    o.init_macro(*lbgen.rt_macro(lx_total, ly, T0, lx=probe_w))
    t = time.perf_counter()
    o.step(1)
    per_site = (time.perf_counter() - t) / (probe_w * ly)
    w = int(max(3, min(lx_total, per_step / (per_site * ly))))
    o = oracle.Lattice(w, ly)
    o.init_macro(*lbgen.rt_macro(lx_total, ly, T0, lx=w))
    o.step(args.warmup)
    t = time.perf_counter()
    o.step(args.steps)
    dt = time.perf_counter() - t
    value = w * ly * args.steps / dt / 1e6
    sample = (f"each step = one full oracle step on columns 0..{w - 1} (all {ly} rows) of the "
              f"{lx_total}x{ly} RT workload")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "MLUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(cfg_name, lx_total, ly, world, args.mode),
        "cpu_baseline": {"value": value, "unit": "MLUPS", "cores": oracle.threads(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(cfg_name, lx_total, ly, world, mode):
    return {"workload": f"D2Q37 fp64 {lx_total}x{ly} lattice, periodic X + thermal walls Y, "
                        f"Rayleigh-Taylor init, {mode} step" + (f", X-slab on {world} GPUs" if world > 1 else ""),
            "name": cfg_name, "lx_total": lx_total, "ly": ly, "sites": lx_total * ly, "mode": mode,
            "parallelism": f"xslab{world}", "l2": "inputs exceed L2 (2 x 1.19 GB/GPU vs 126 MB), no flush",
            "tau": 0.8, "bc_y": "thermal", "init": "isobaric RT (lbgen, seed 1703)"}


def kernel_passes(lb, lx_total, ly, fields, hbm_peak, fp64_peak, ncu, nsteps=10):
    """Per-kernel CUDA-event times of split BGK, fused regularised and split
    regularised steps on the same workload (library instrumentation)."""
    kern = {}
    for mode, coll, impl in (("split", "bgk", "ldg"), ("split", "bgk", "tma"), ("fused", "bgk", "tma"),
                             ("fused", "regularized", "ldg"), ("split", "regularized", "ldg"), ("fused", "bgk", "ldg"),
                             ("fused", "regularized", "tb")):
        # "tb": the two-step kernel (the default path); the others pin the one-step kernels
        g = lb.Lattice(lx_total, ly, mode=mode, collision=coll, temporal=(impl == "tb"))
        if mode == "split":
            g.set_propagate_impl(impl)
        elif impl != "tb":
            g.set_fused_impl(impl)
        g.init_macro(*fields)
        g.step(3)
        g.profile(True)
        g.profile_reset()
        g.step(nsteps)
        sp = g.profile_read()
        g.close()
        for k, v in sp.items():
            if k in kern:
                continue
            avg = v["total_ms"] / max(1, v["launches"])
            e = {"avg_ms": avg, "launches": v["launches"]}
            if k in ("k_propagate", "k_propagate_tma", "k_collide", "k_collide_reg", "k_step_fused_reg",
                     "k_step_fused_tma"):
                per = BYTES_PER_SITE * v["units"] / v["launches"]
                e["gbs"] = per / (avg * 1e-3) / 1e9
                e["hbm_frac"] = e["gbs"] / hbm_peak
                e["mlups"] = v["units"] / v["launches"] / (avg * 1e-3) / 1e6
            if k in ("k_collide", "k_collide_reg", "k_step_fused_reg"):
                fl = ncu.get("kernels", {}).get(k, {}).get("flops_per_site")
                if fl and fp64_peak:
                    tf = fl * e["mlups"] * 1e6 / 1e12
                    e.update({"flops_per_site_ncu": fl, "fp64_tflops": tf, "fp64_frac": tf / fp64_peak,
                              "fp64_peak_tflops": fp64_peak})
                e["paper_convention_6500_flop_tflops"] = 6500 * e["mlups"] * 1e6 / 1e12
            if k.startswith("k_step2_tb"):
                # one launch = two time steps; algorithmic HBM traffic = one read + one
                # write of the state (592 B/site) per launch
                e["site_updates_per_launch"] = v["units"] / v["launches"]
                e["mlups"] = v["units"] / v["launches"] / (avg * 1e-3) / 1e6
                e["gbs"] = BYTES_PER_SITE * v["units"] / 2 / v["launches"] / (avg * 1e-3) / 1e9
                e["hbm_frac"] = e["gbs"] / hbm_peak
            kern[k] = e
        step_ms = sum(v["total_ms"] for v in sp.values()) / nsteps
        kern[f"{mode}_{coll}" + ("_" + impl if impl in ("tma", "tb") else "") + "_step_mlups"] = \
            lx_total * ly / (step_ms * 1e-3) / 1e6
    return kern


# ----------------------------------------------------------------------------- our leg

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="weak1920", choices=sorted(CONFIGS))
    ap.add_argument("--mode", default="fused", choices=["fused", "split"])
    ap.add_argument("--overlap", type=int, default=-1, help="-1: auto (on for N>1)")
    ap.add_argument("--transport", default="auto", choices=["auto", "peer", "nccl"],
                    help="N>1 halo exchange: peer stores fused into the step kernel (CUDA IPC over "
                         "NVLink, default) or NCCL send/recv on a comm stream overlapped with the bulk")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / split pass / cpu baseline")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    lx_cfg, ly, scaling = CONFIGS[args.config]
    lx_total = lx_cfg * world if scaling == "weak" else lx_cfg

    if args.impl == "reference":
        run_reference(args, args.config, lx_total, ly, scaling, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    import lbgen
    import paper_1703_00186_b200 as lb
    from paper_1703_00186_b200 import perfmodel as pm

    # LB_BENCH_SAME_GPU=1 (test only): all ranks on cuda:0, gloo process group,
    # no NCCL communicator, peer transport -- exercises the N > 1 code path of
    # this script on a one-GPU box (numbers meaningless: ranks time-slice).
    same_gpu = os.environ.get("LB_BENCH_SAME_GPU") == "1" and world > 1
    dev_index = 0 if same_gpu else local_rank
    torch.cuda.set_device(dev_index)
    if world > 1 and same_gpu:
        dist.init_process_group("gloo")
        nccl_id = None
    elif world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        obj = [lb.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        nccl_id = None
    overlap = (world > 1) if args.overlap < 0 else bool(args.overlap)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if same_gpu else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    T0 = lb.t0()
    g = lb.Lattice(lx_total, ly, mode=args.mode, overlap=overlap, rank=rank, nranks=world, nccl_id=nccl_id)
    transport = "local" if world == 1 else ("nccl" if args.transport == "nccl" or args.mode != "fused" else "peer")
    lx = g.lx
    fields = lbgen.rt_macro(lx_total, ly, T0, x0=rank * lx, lx=lx)
    g.init_macro(*fields)
    if transport == "peer":
        try:
            g.set_peers_ipc()
        except Exception as exc:  # fall back to the NCCL ring (communicator exists)
            if same_gpu:
                raise
            print(f"peer exchange unavailable ({exc}); using NCCL", file=sys.stderr)
            transport = "nccl"
    barrier()
    stream = torch.cuda.current_stream()

    # ---- warm-up, then exactly K timed steps (device time, max over ranks).
    # The headline region carries no per-launch events (they cost ~1 % of a
    # step); the dominant kernel's launch durations are measured live in a
    # second timed region of K steps right after it, with the library's
    # per-launch CUDA events on the launch stream.
    g.step(args.warmup)
    g.sync()
    launches0 = g.launch_count()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev_index) as clk:   # thread started before the region, samples counted within it
        time.sleep(0.005)
        clk.begin()
        e0.record(stream)
        g.step(args.steps)
        e1.record(stream)
        g.sync()
        torch.cuda.synchronize()
        clk.end()
    barrier()
    launches = g.launch_count() - launches0
    ms = max_over_ranks(e0.elapsed_time(e1))
    # ---- the dominant kernel's launch durations (CUDA events per launch on the
    # launch stream), right after the headline region, after one idle second:
    # a sustained run of the two-step kernel reaches the board's power limit
    # within ~1 s and the SM clock falls (DESIGN.md §6 "Power"); an idle second
    # restores it, so this region starts from the headline's power state
    # instead of inheriting the heat of the headline region
    time.sleep(1.0)
    g.profile(True)
    g.profile_reset()
    barrier()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    g.step(args.steps)
    e3.record(stream)
    g.sync()
    prof = g.profile_read()
    g.profile(False)
    ms_prof = e2.elapsed_time(e3)
    # ---- spread (median over >= 5 repetitions): 5 more timed
    # regions of max(K, 200) steps each, same protocol; the headline value
    # stays the contract's region above
    k_rep = max(args.steps, 200) // 2 * 2
    reps = []
    for _ in range(5):
        barrier()
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record(stream)
        g.step(k_rep)
        r1.record(stream)
        g.sync()
        torch.cuda.synchronize()
        reps.append(pm.mlups(lx_total * ly * k_rep, max_over_ranks(r0.elapsed_time(r1)) * 1e-3))
    sites_all = lx_total * ly
    value = pm.mlups(sites_all * args.steps, ms * 1e-3)   # Table 1 convention (tests/test_metrics.py)

    peaks = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"), {}) or {}
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (driver-measured copy)"
    if not hbm_peak:
        hbm_peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    ncu = load_json(os.path.join(ROOT, "profiles", "ncu_summary.json"), {}) or {}
    fp64 = (load_json(os.path.join(ROOT, "profiles", "r02_fp64_hbm_microbench.json"), {})
            or load_json(os.path.join(ROOT, "profiles", "r01_fp64_hbm_microbench.json"), {}) or {})
    fp64_peak = fp64.get("fp64_tflops")   # measured DFMA peak (tools/fp64_bench.py, NVML-sampled clock)

    # dominant kernel: the two-step kernel k_step2_tb (the default N = 1 path),
    # else every launch of k_step_fused (whole lattice, or bulk + border
    # launches of the overlapped schedule), aggregated
    two_step = "k_step2_tb" in prof
    kname = "k_step2_tb" if two_step else "k_step_fused"
    parts = [v for k, v in prof.items() if k == kname] if two_step else \
        [v for k, v in prof.items() if k.startswith("k_step_fused") and "_reg" not in k]
    fk = {"launches": sum(v["launches"] for v in parts), "total_ms": sum(v["total_ms"] for v in parts),
          "units": sum(v["units"] for v in parts)} if parts else None
    if fk and world > 1:
        # bulk and border launches differ in size: use steps as the launch unit
        fk["launches"] = args.steps
    roofline = None
    # the headline region itself, when it launched nothing but the dominant
    # kernel (N = 1, two-step kernel, K even: K / 2 launches): its events give
    # the kernel's average launch duration directly, including the overlap of
    # consecutive launches (programmatic dependent launch), which the per-launch
    # events of the second region (they sit between launches) prevent
    only_dominant = (two_step and world == 1 and set(prof) == {kname} and launches > 0
                     and int(launches) == args.steps // 2 and args.steps % 2 == 0)
    if fk and fk["launches"]:
        event_avg_ms = fk["total_ms"] / fk["launches"]
        avg_ms = ms / launches if only_dominant else event_avg_ms
        # algorithmic bytes of one launch: one read + one write of the state
        # (592 B/site) -- per step for k_step_fused, per TWO steps for
        # k_step2_tb (its units are site updates: 2 x sites per launch)
        sites_per_launch = fk["units"] / fk["launches"] / (2 if two_step else 1)
        bytes_per_launch = BYTES_PER_SITE * sites_per_launch
        achieved = pm.gbs(sites_per_launch, avg_ms * 1e-3)   # sites x 592 B / t
        kn = ncu.get("kernels", {}).get(kname, {})
        traffic = kn.get("dram_bytes_per_site")
        roofline = {"kernel": kname, "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                    "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                    "traffic": (traffic * sites_per_launch) if traffic else None,
                    "algorithmic_bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                    "event_avg_launch_ms": event_avg_ms,
                    "share_of_step": fk["total_ms"] / ms_prof,
                    "measured": ("CUDA events on the launch stream around the headline region, which launched "
                                 f"only {kname} ({int(launches)} launches; region time / launches); "
                                 "event_avg_launch_ms: per-launch events over a second region of the same "
                                 f"{args.steps} steps (they serialise the launches) -- share_of_step from it")
                                if only_dominant else
                                ("per-launch CUDA events on the launch stream over a second timed region "
                                 f"of the same {args.steps} steps"),
                    "peak_source": peak_src,
                    "traffic_source": ncu.get("source") if traffic else None}
        fl = kn.get("flops_per_site")   # ncu FP64 flops per site per launch (FMA = 2)
        if fl and fp64_peak:
            # the collisions' FP64 rate inside the dominant kernel (BASELINE's "collide
            # FP64 % of peak"): not its bound, reported beside the HBM roofline
            tf = fl * sites_per_launch / (avg_ms * 1e-3) / 1e12
            roofline["fp64"] = {"flops_per_site_per_launch": fl, "tflops": round(tf, 2),
                                "peak_tflops": fp64_peak, "frac": round(tf / fp64_peak, 4)}
        if two_step:
            roofline["steps_per_launch"] = 2
            roofline["one_step_equivalent_gbs"] = round(2 * achieved, 1)
            roofline["note"] = ("two time steps per HBM pass (temporal blocking): achieved/frac count the "
                                "592 B/site one pass moves; one_step_equivalent_gbs is the bandwidth a "
                                "one-step kernel would need for the same MLUPS (DESIGN.md section 6)")

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "MLUPS", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args.config, lx_total, ly, world, args.mode),
        "clocks": clk.summary(), "gpu_launches": int(launches),
        "repetitions": {"regions": len(reps), "steps_each": k_rep, "median": round(statistics.median(reps), 2),
                        "min": round(min(reps), 2), "max": round(max(reps), 2), "unit": "MLUPS"},
        "roofline": roofline,
        "kernel_times_ms": {k: {"avg_ms": v["total_ms"] / max(1, v["launches"]), "launches": v["launches"]}
                            for k, v in prof.items()},
    }
    line["config"]["overlap"] = overlap
    line["config"]["transport"] = transport
    if same_gpu:
        line["config"]["same_gpu_test"] = "all ranks on cuda:0 (test of the N>1 code path, not a measurement)"

    if not args.no_extras:
        # ---- e2e through the C ABI with pinned host buffers (same fused path)
        state_bytes = 37 * g.sites * 8
        host_in = torch.empty(37 * g.sites, dtype=torch.float64).pin_memory()
        host_out = torch.empty((37, lx_total, ly), dtype=torch.float64).pin_memory() if rank == 0 else None
        g.init_macro(*fields)
        st0 = g.peek(0)
        host_in.numpy()[:] = st0.reshape(-1)
        del st0
        # a user's run: upload once, K steps with one result per step read
        # back, gather once.  K = max(timed K, 1000): at the driver's K = 20 the
        # two 1.17 GB PCIe copies alone would be ~90 % of the region
        # (e2e_at_timed_K below repeats it at the timed K for transparency)
        k_e2e = max(args.steps, 1000) // 2 * 2
        g.monitor(True)   # per-step invariants reduced inside the step kernel (lb_monitor)
        mon = torch.empty((k_e2e, 5), dtype=torch.float64).pin_memory()   # per-step results on the host
        # the two-step kernel (default at N = 1 with walls) carries monitors of
        # BOTH its states: lb_step(2) + lb_invariants_pair_async still returns
        # one result per time step
        pair = False
        try:
            g.step(2)
            g.invariants_pair_async(mon[0:2])
            g.sync()
            pair = True
        except lb.LBError:
            pass
        barrier()
        torch.cuda.synchronize()
        t = time.perf_counter()
        g.set_state(host_in.numpy())
        barrier()  # peer mode: neighbours' states set before the first halo pull
        if pair:
            for k in range(0, k_e2e, 2):
                g.step(2)
                g.invariants_pair_async(mon[k:k + 2])   # D2H of both steps' results into pinned memory
        else:
            for k in range(k_e2e):
                g.step(1)
                g.invariants_async(mon[k])   # D2H of the step's result into pinned memory
        if same_gpu:
            g.peek(0)   # no communicator: each rank reads its own slab back
        else:
            g.gather(out=host_out.numpy() if host_out is not None else None)   # synchronising
        e2e_s = max_over_ranks(time.perf_counter() - t)
        m = mon.numpy()
        if world > 1:
            # (after the timed region) the per-step results are this rank's
            # slab (lb_invariants_pair_async is not collective): sum over ranks
            dev = "cpu" if same_gpu else "cuda"
            sums = torch.from_numpy(m[:, :4].copy()).to(dev)
            mins = torch.from_numpy(m[:, 4].copy()).to(dev)
            dist.all_reduce(sums, op=dist.ReduceOp.SUM)
            dist.all_reduce(mins, op=dist.ReduceOp.MIN)
            m = np.concatenate([sums.cpu().numpy(), mins.cpu().numpy()[:, None]], axis=1)
        mass_drift = float(abs(m[-1, 0] - m[0, 0]) / m[0, 0])
        line["e2e"] = {"value": round(sites_all * k_e2e / e2e_s / 1e6, 2), "unit": "MLUPS",
                       "h2d_bytes_per_step": state_bytes / k_e2e,
                       "d2h_bytes_per_step": (state_bytes + 5 * 8 * k_e2e) / k_e2e,
                       "steps": k_e2e, "mode": args.mode,
                       "timed": ("lb_set_state(pinned host) + K/2 x (lb_step(2) on the two-step kernel with "
                                 "monitors of both states + lb_invariants_pair_async -> pinned host: one result "
                                 "per step) + lb_gather(pinned host)") if pair else
                                ("lb_set_state(pinned host) + K x (lb_step(1) with fused monitors + "
                                 "lb_invariants_async -> pinned host) + lb_gather(pinned host)"),
                       "per_step_results_ok": bool(np.isfinite(m).all() and (m[:, 4] > 0).all()),
                       "mass_drift_over_K": mass_drift}
        if k_e2e != args.steps // 2 * 2 and args.steps >= 2:
            k2 = args.steps // 2 * 2
            barrier()
            torch.cuda.synchronize()
            t = time.perf_counter()
            g.set_state(host_in.numpy())
            barrier()
            for k in range(0, k2, 2 if pair else 1):
                if pair:
                    g.step(2)
                    g.invariants_pair_async(mon[k:k + 2])
                else:
                    g.step(1)
                    g.invariants_async(mon[k])
            if same_gpu:
                g.peek(0)
            else:
                g.gather(out=host_out.numpy() if host_out is not None else None)
            dt2 = max_over_ranks(time.perf_counter() - t)
            line["e2e_at_timed_K"] = {"value": round(sites_all * k2 / dt2 / 1e6, 2), "unit": "MLUPS", "steps": k2,
                                      "h2d_bytes_per_step": state_bytes / k2,
                                      "d2h_bytes_per_step": (state_bytes + 5 * 8 * k2) / k2}
        del host_in, host_out
        # ---- per-kernel passes (N = 1): split BGK (propagate GB/s, collide FP64 %),
        #      fused and split regularised collide (NEXT 1)
        if world == 1:
            g.close()
            del g
            torch.cuda.empty_cache()
            line["kernels"] = kernel_passes(lb, lx_total, ly, fields, hbm_peak, fp64_peak, ncu)
        # ---- CPU oracle baseline (rank 0, N = 1 only)
        if world == 1 and rank == 0:
            mlups, cores, sample, dt, w, ns = oracle_throughput(lx_total, ly,
                                                                float(os.environ.get("LB_CPU_BUDGET_S", "15")))
            line["cpu_baseline"] = {"value": round(mlups, 3), "unit": "MLUPS", "cores": cores,
                                    "kind": "oracle", "sample": sample}
            if os.environ.get("LB_CPU_PROTOCOL", "1") == "1":
                line["cpu_baseline"]["protocol"] = oracle_protocol()

    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
