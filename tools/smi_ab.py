"""Does nvidia-smi sampling slow the timed region?  config 5 (heat SDO4 1024^3) and config 4
(PW set) timed for 400 steps with no sampler, with `nvidia-smi -lms 100` and with `-lms 500`
running, interleaved, CUDA events on the launching stream.

  python tools/smi_ab.py [rounds]
"""
import ctypes
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
QUERY = ["nvidia-smi", "-i", "0",
         "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
         "--format=csv,noheader,nounits"]


def timed(plan, steps, period):
    proc = None
    if period:
        proc = subprocess.Popen(QUERY + ["-lms", str(period)], stdout=subprocess.DEVNULL,
                                stderr=subprocess.DEVNULL)
        time.sleep(1.0)  # sampler live
    plan.run(steps, stream=sh)  # keep the GPU busy up to the timed region
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    plan.run(steps, stream=sh)
    e1.record(s)
    torch.cuda.synchronize()
    if proc:
        proc.terminate()
        proc.wait()
    return e0.elapsed_time(e1) / steps


for name, prog in (("heat3d_1024", hg.build_kernel(hg.KernelSpec("heat", 3, 1024, 4, "f32"))),
                   ("pw_advection", hg.Program.pw_advection(128, 512, 512))):
    plan = hg.Plan(prog)
    plan.init_fields(stream=sh)
    plan.run(20, stream=sh)
    res = {}
    for r in range(rounds):
        for period in (0, 100, 500):
            res.setdefault(period, []).append(timed(plan, 400, period))
    for period, v in res.items():
        print(f"{name} sampler={period or 'off'} ms/step " + " ".join(f"{x:.4f}" for x in v),
              flush=True)
    plan.close()
