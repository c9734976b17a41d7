"""Burst vs sustained rate under the power cap: a STREAM-style copy (torch, the MEASURED_PEAKS
recipe), config 5 heat and config 4 PW, each run back to back for ~3 s in ~20 ms chunks timed
with CUDA events, with nvidia-smi sampling SM clock and power every 100 ms.

  python tools/sustain_probe.py [seconds]
"""
import ctypes
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)


class Smi:
    def __enter__(self):
        self.lines = []
        self.p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw",
                                   "--format=csv,noheader,nounits", "-lms", "100"],
                                  stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.t = threading.Thread(target=lambda: [self.lines.append((time.time(), ln))
                                                  for ln in self.p.stdout], daemon=True)
        self.t.start()
        time.sleep(1.0)
        return self

    def __exit__(self, *a):
        self.p.terminate()
        self.p.wait()


def probe(name, step, bytes_per_step, per_chunk):
    time.sleep(2.0)  # idle: let the power state settle between workloads
    with Smi() as smi:
        t_start = time.time()
        rates = []
        while time.time() - t_start < secs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            step(per_chunk)
            e1.record(s)
            e1.synchronize()
            rates.append(bytes_per_step * per_chunk / (e0.elapsed_time(e1) / 1e3) / 1e9)
        samples = [ln.split(",") for t, ln in smi.lines if t >= t_start]
    clk = [float(a) for a, b in samples if a.strip().replace(".", "").isdigit()]
    pw = [float(b) for a, b in samples if b.strip().replace(".", "").isdigit()]
    n = len(rates)
    first = rates[:max(1, n // 20)]
    last = rates[n // 2:]
    print(f"{name}: first {len(first)} chunks {sum(first) / len(first):.0f} GB/s, max "
          f"{max(rates):.0f}; second half {sum(last) / len(last):.0f} GB/s; SM MHz "
          f"{min(clk) if clk else 0:.0f}-{max(clk) if clk else 0:.0f} "
          f"(median {sorted(clk)[len(clk) // 2] if clk else 0:.0f}); power W median "
          f"{sorted(pw)[len(pw) // 2] if pw else 0:.0f} max {max(pw) if pw else 0:.0f}",
          flush=True)


a = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
b = torch.empty_like(a)
a.fill_(1.0)


def copy(k):
    for _ in range(k):
        b.copy_(a)


probe("copy 4 GiB", copy, 2 * a.numel() * 4, 10)
del a, b
torch.cuda.empty_cache()
for name, prog, bpp, chunk in (
        ("heat3d SDO4 1024^3", hg.build_kernel(hg.KernelSpec("heat", 3, 1024, 4, "f32")), 8, 14),
        ("PW set 128x512x512", hg.Program.pw_advection(128, 512, 512), 24, 130)):
    plan = hg.Plan(prog)
    plan.init_fields(stream=sh)
    plan.run(10, stream=sh)
    probe(name, lambda k: plan.run(k, stream=sh), bpp * prog.core_points(), chunk)
    plan.close()
