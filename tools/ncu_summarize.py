"""Summarise an ncu --metrics CSV (tools/gpu_bench_round.sh) into
profiles/ncu_summary.json: per kernel, mean over launches of DRAM bytes per
site, FP64 flops per site (2*DFMA + DADD + DMUL), FP64-pipe %, DRAM % and time.

usage: python tools/ncu_summarize.py <ncu_metrics.csv> <sites> <out.json> [label]
"""
import collections
import csv
import json
import sys

path, sites, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
label = sys.argv[4] if len(sys.argv) > 4 else path
rows = list(csv.reader(open(path)))
hdr = None
per = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) < len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].replace("(anonymous namespace)::", "").replace("unnamed>::", "").split("(")[0].replace("void ", "")
    base = name.split("<")[0]
    targs = name[len(base):].strip("<>").replace(" ", "").split(",") if "<" in name else []
    # collision kind: k_step_fused<BC, COLL, MON> / k_collide<COLL>
    coll_arg = {"k_step_fused": 1, "k_collide": 0, "k_step2_tb": 0}.get(base)
    if coll_arg is not None and len(targs) > coll_arg and targs[coll_arg] == "1":
        base += "_reg"
    if base.startswith("k_step_fused") and len(targs) > 2 and targs[2] in ("1", "true"):
        base += "_mon"
    try:
        v = float(d["Metric Value"].replace(",", ""))
    except ValueError:
        continue
    per[(base, d["ID"])][d["Metric Name"]] = v
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for (base, _), m in per.items():
    for k, v in m.items():
        agg[base][k].append(v)
res = {"source": label, "sites": sites, "kernels": {}}
for base, m in agg.items():
    mean = {k: sum(v) / len(v) for k, v in m.items()}
    e = {"launches": len(next(iter(m.values())))}
    if "dram__bytes_read.sum" in mean:
        e["dram_bytes_per_launch"] = mean["dram__bytes_read.sum"] + mean["dram__bytes_write.sum"]
        e["dram_bytes_per_site"] = e["dram_bytes_per_launch"] / sites
    if "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum" in mean:
        fl = (2 * mean["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
              + mean["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
              + mean["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])
        e["flops_per_launch"] = fl
        e["flops_per_site"] = fl / sites
    for k, short in [("gpu__time_duration.sum", "time_ns"),
                     ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
                     ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_of_peak"),
                     ("launch__registers_per_thread", "registers"),
                     ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct")]:
        if k in mean:
            e[short] = mean[k]
    res["kernels"][base] = e
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
