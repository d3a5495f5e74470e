"""Summarise an ncu --set full report of k_step2_tb: headline metrics, warp
stall reasons per issued instruction, stall samples by SASS opcode and the top
stalled instructions (measurement tool; reads .ncu-rep files with ncu -i).

python tools/ncu_stalls.py REPORT.ncu-rep [REPORT2 ...] > profiles/r02_tb_ncu_stalls.json
"""
import csv
import io
import json
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_active.avg",
        "sm__cycles_active.max", "sm__cycles_active.min", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    r = ncu_csv(rep, "raw")
    hdr, vals = r[0], r[2]
    raw = dict(zip(hdr, vals))
    res = {"report": rep, "metrics": {k: raw.get(k) for k in KEYS}}
    res["stalls_per_issue"] = {h.split("issue_stalled_")[1].split("_per_issue")[0]: round(float(v), 3)
                               for h, v in raw.items()
                               if "average_warps_issue_stalled" in h and "per_issue_active" in h and float(v) > 0.01}
    rows = ncu_csv(rep, "source", ["--print-source", "sass"])
    h, data = rows[1], rows[2:]
    iS, iW = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[iW]) for x in data)
    by_op = Counter()
    for x in data:
        t = x[iS].split()
        op = (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")).split(".")[0]
        by_op[op] += int(x[iW])
    res["stall_samples_by_opcode_pct"] = {k: round(100 * v / tot, 1) for k, v in by_op.most_common(12)}
    cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
    top = sorted(data, key=lambda x: -int(x[iW]))[:8]
    res["top_stalled_instructions"] = [
        {"sass": x[iS].strip()[:60], "pct": round(100 * int(x[iW]) / tot, 1),
         "reasons": dict(sorted(((c[6:], int(x[h.index(c)])) for c in cols if x[h.index(c)] not in ("", "0")),
                                key=lambda kv: -kv[1])[:3])} for x in top]
    return res


if __name__ == "__main__":
    print(json.dumps([summarise(r) for r in sys.argv[1:]], indent=1))
