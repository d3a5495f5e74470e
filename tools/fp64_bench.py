"""FP64 DFMA peak + HBM copy microbenchmark with NVML clock samples
(SURVEY §8d "FP64 peak microbenchmark"; measurement tool, GPU box only).

    python tools/fp64_bench.py [--reps 120] [--out profiles/r02_fp64_hbm_microbench.json]

Builds tools/fp64_peak.cu (sm_100a), runs it while a thread samples the SM
clock and throttle reasons every 5 ms, and reports the measured FP64 rate
next to 148 SM x 64 DFMA/clk x 2 flop x the sampled clock.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=120)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    src = os.path.join(ROOT, "tools", "fp64_peak.cu")
    exe = os.path.join(ROOT, "tools", "fp64_peak")
    if not os.path.exists(exe) or os.path.getmtime(exe) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-o", exe, src])
    with ClockSampler(0) as clk:
        out = subprocess.run([exe, str(a.reps)], capture_output=True, text=True, check=True).stdout
    res = json.loads(out.strip().splitlines()[-1])
    c = clk.summary()
    res["clocks_during_run"] = c
    if c.get("sm_mhz"):
        res["fp64_peak_at_sampled_clock_tflops"] = round(148 * 64 * 2 * c["sm_mhz"] * 1e6 / 1e12, 2)
        res["fp64_frac_of_clock_peak"] = round(res["fp64_tflops"] / res["fp64_peak_at_sampled_clock_tflops"], 4)
    res["what"] = ("dfma_chains<8>: 148 x 8 blocks of 256 threads, 8 independent fma(x, y, x) chains per thread, "
                   "2^16 iterations, best of --reps launches; copy_v2: double2 grid-stride copy of 2 GiB, best of 10; "
                   "NVML SM clock sampled every 5 ms over the whole run")
    js = json.dumps(res, indent=1)
    if a.out:
        open(a.out, "w").write(js + "\n")
    print(js)


if __name__ == "__main__":
    main()
