"""Small driver for ncu captures: N time steps of one star plan (no dmp, no e2e)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--kind", default="heat")
ap.add_argument("--extent", type=int, default=1024)
ap.add_argument("--order", type=int, default=4)
ap.add_argument("--rank", type=int, default=3)
ap.add_argument("--steps", type=int, default=6)
ap.add_argument("--chunks", type=int, default=0)
a = ap.parse_args()
prog = hg.build_kernel(hg.KernelSpec(a.kind, a.rank, a.extent, a.order, "f32"))
plan = hg.Plan(prog)
plan.init_fields()
plan.set_tuning(a.chunks)
plan.run(a.steps)
plan.download(0)
print("ok", plan.kernel_name)
