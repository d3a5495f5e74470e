"""Does the two-step kernel slow down over a long run, and why (tools only)?

Times consecutive 200-step chunks of lb_step at 1920x2048 for ~4000 steps,
then re-uploads the initial state and times one more chunk: a slowdown that
stays after the re-upload is the device (clocks, power, temperature), one that
goes away is the data.  Clocks and power are sampled with NVML per chunk.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import lbgen  # noqa: E402
import paper_1703_00186_b200 as lbm  # noqa: E402

try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
except Exception:  # noqa: BLE001
    h = None


def nv():
    if h is None:
        return {}
    return {"sm_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
            "mem_mhz": pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
            "power_w": pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
            "temp_c": pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)}


lx, ly = 1920, 2048
coll = sys.argv[1] if len(sys.argv) > 1 else "bgk"
s = torch.cuda.Stream()
g = lbm.Lattice(lx, ly, collision=coll, stream=s)
fields = lbgen.rt_macro(lx, ly, 1.0 / 1.19697977039307435897239 ** 2)
g.init_macro(*fields)
st0 = g.gather()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def chunk(tag, k=200):
    with torch.cuda.stream(s):
        e0.record(s)
        g.step(k)
        e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / k
    print(json.dumps({"chunk": tag, "ms_per_step": round(ms, 5), "mlups": round(lx * ly / ms / 1e3, 1), **nv()}),
          flush=True)


for c in range(20):
    chunk(c)
g.set_state(st0)
g.sync()
chunk("reupload")
torch.cuda.synchronize()
torch.cuda._sleep(int(2e9))  # ~1 s idle
torch.cuda.synchronize()
chunk("after_idle")
