"""Star tile geometry A/B on the local shapes of the strong-scaling grids (heat SDO4 f32):
the 64x16 tile (GEO 0) against the 128x12 tile (GEO 1), CUDA events, steady state.

  python tools/geo_ab.py
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

SHAPES = [(2048, 2048, 512), (2048, 1024, 1024), (1024, 2048, 1024), (1024, 1024, 2048),
          (2048, 512, 2048), (1024, 1024, 1024), (512, 512, 512)]
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
for shape in SHAPES:
    res = []
    for geo in ("0", "1"):
        os.environ["HG_STAR_GEO"] = geo
        prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents(list(shape))
        plan = hg.Plan(prog)
        plan.init_fields(stream=sh)
        plan.run(6, stream=sh)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = max(10, int(2e10 / prog.core_points()))
        torch.cuda.synchronize()
        e0.record(s)
        plan.run(steps, stream=sh)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        res.append((geo, ms, prog.core_points() / ms / 1e6))
        plan.close()
    print(shape, " ".join(f"geo{g}: {ms:.3f} ms {gp:.1f} GPts/s" for g, ms, gp in res), flush=True)
