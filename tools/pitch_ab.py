"""Row-pitch padding A/B (HG_PITCH_PAD extra 128-byte lines per row) for the heat SDO4 star
kernel on a few shapes, CUDA events, steady state."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

SHAPES = [(1024, 1024, 1024), (512, 512, 512), (2048, 512, 2048), (2048, 2048, 512)]
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
for shape in SHAPES:
    out = []
    for pad in ("0", "1", "2", "3", "4"):
        os.environ["HG_PITCH_PAD"] = pad
        prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents(list(shape))
        plan = hg.Plan(prog)
        plan.init_fields(stream=sh)
        plan.run(6, stream=sh)
        steps = max(10, int(2e10 / prog.core_points()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        plan.run(steps, stream=sh)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out.append(f"pad{pad} {prog.core_points() / ms / 1e6:.1f}")
        name = plan.kernel_name
        plan.close()
    print(shape, name, " ".join(out), flush=True)
