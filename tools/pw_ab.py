"""Fused-apply A/B on BASELINE config 4 (PW advection set, 128 x 512 x 512 f32): one CTA per
unit against persistent CTAs (HG_JIT_PERSIST), packed against scalar adds (HG_JIT_PACK), and
z-chunk counts, interleaved rounds,
CUDA events on the launching stream, steady state.

  python tools/pw_ab.py [rounds]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402

PEAK = 6451.8  # GB/s, MEASURED_PEAKS.json
BYTES = 24  # 3 fields read + 3 written, f32, per point
VARIANTS = [("1", 0, "1"), ("1", 0, "0"), ("0", 0, "0"), ("1", 16, "1")]  # (HG_JIT_PERSIST, chunks, HG_JIT_PACK)
rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
s = torch.cuda.current_stream()
sh = ctypes.c_void_p(s.cuda_stream)
prog = hg.Program.pw_advection(128, 512, 512)
pts = prog.core_points()
plans = {}
for persist, chunks, pack in VARIANTS:
    os.environ["HG_JIT_PERSIST"] = persist
    os.environ["HG_JIT_PACK"] = pack
    plan = hg.Plan(prog)
    plan.set_tuning(chunks=chunks)
    plan.init_fields(stream=sh)
    plan.run(20, stream=sh)
    plans[(persist, chunks, pack)] = plan
torch.cuda.synchronize()
best = {}
for r in range(rounds):
    for key, plan in plans.items():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        steps = 400
        e0.record(s)
        plan.run(steps, stream=sh)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        best.setdefault(key, []).append(ms)
for (persist, chunks, pack), v in best.items():
    ms = min(v)
    print(f"persist={persist} pack={pack} chunks={chunks or 'auto'}: {ms * 1e3:.1f} us/step "
          f"{pts / ms / 1e6:.1f} GPts/s frac {pts * BYTES / ms / 1e6 / PEAK:.3f} "
          f"(rounds: {' '.join(f'{x * 1e3:.1f}' for x in v)})", flush=True)
ref = None
for key, plan in plans.items():
    outs = [plan.download(b) for b in range(prog.nfields)]
    if ref is None:
        ref = outs
    assert all((o.view("u4") == r.view("u4")).all() for o, r in zip(outs, ref)), key
    plan.close()
print("all fields bitwise equal across variants")
