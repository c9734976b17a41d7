"""Kernel timing sweep (CUDA events, no profiler): GPts/s and algorithmic GB/s per workload.

  HG_LIB=<variant .so> python tools/sweep.py [--quick]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

WL = [  # name, spec, bytes/pt, steps
    ("heat3d_so4_1024", ("heat", 3, 1024, 4), 8, 60),
    ("heat3d_so4_512", ("heat", 3, 512, 4), 8, 200),
    ("wave3d_so8_1024", ("wave", 3, 1024, 8), 12, 40),
    ("heat3d_so2_1024", ("heat", 3, 1024, 2), 8, 60),
    ("heat3d_so8_1024", ("heat", 3, 1024, 8), 8, 60),
    ("heat2d_so2_1024", ("heat", 2, 1024, 2), 8, 2000),
    ("heat2d_so2_16384", ("heat", 2, 16384, 2), 8, 60),
    ("pw_advection_128x512x512", "pw", 24, 100),
]


def main():
    chunks = [int(x) for x in os.environ.get("HG_CHUNKS", "0").split(",")]
    only = os.environ.get("HG_ONLY")
    s = torch.cuda.current_stream()
    sh = hg.C.c_void_p(s.cuda_stream) if hasattr(hg, "C") else None
    import ctypes
    sh = ctypes.c_void_p(s.cuda_stream)
    res = {}
    for name, spec, bpp, steps in WL:
        if only and name not in only.split(","):
            continue
        prog = (hg.Program.pw_advection(128, 512, 512) if spec == "pw"
                else hg.build_kernel(hg.KernelSpec(*spec, "f32")))
        plan = hg.Plan(prog)
        plan.init_fields(stream=sh)
        for ch in chunks:
            plan.set_tuning(ch)
            plan.run(5, stream=sh)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            plan.run(steps, stream=sh)
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / steps
            pts = prog.core_points()
            res[f"{name}/c{ch}"] = {"ms": ms, "gpts": pts / ms / 1e6,
                                    "gbs": pts * bpp / ms / 1e6}
            print(f"{name:20s} chunks={ch:3d} {ms*1e3:9.1f} us  {pts/ms/1e6:7.1f} GPts/s "
                  f"{pts*bpp/ms/1e6:7.0f} GB/s", flush=True)
        plan.close()
    print("JSON", json.dumps(res))


if __name__ == "__main__":
    main()
