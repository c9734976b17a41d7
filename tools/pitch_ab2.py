"""Row-pitch padding sweep (HG_PITCH_PAD) over the benched and strong-scaling rank shapes."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

CASES = [("heat", 4, (1024, 1024, 1024)), ("wave", 8, (1024, 1024, 1024)),
         ("heat", 4, (1024, 1024, 2048)), ("heat", 4, (1024, 2048, 2048)),
         ("heat", 4, (768, 768, 768)), ("heat", 4, (1024, 1024, 1536)),
         ("heat", 4, (1024, 1024, 1000)), ("heat", 4, (512, 512, 512)),
         ("heat", 4, (512, 2048, 1024))]
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
for kind, order, shape in CASES:
    out = []
    for pad in ("0", "1", "2"):
        os.environ["HG_PITCH_PAD"] = pad
        prog = hg.build_kernel(hg.KernelSpec(kind, 3, 8, order, "f32")).with_extents(list(shape))
        plan = hg.Plan(prog)
        plan.init_fields(stream=sh)
        plan.run(6, stream=sh)
        steps = max(8, int(1.5e10 / prog.core_points()))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        plan.run(steps, stream=sh)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        pitch = plan.layout(0).pitch
        out.append(f"pad{pad}(pitch {pitch}) {prog.core_points() / ms / 1e6:.1f}")
        plan.close()
    print(kind, shape, " ".join(out), flush=True)
