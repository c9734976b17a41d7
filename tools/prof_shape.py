"""ncu helper: heat3d SDO4 star kernel on an arbitrary (nz, ny, nx) core."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg
ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="1024,1024,1024")
ap.add_argument("--chunks", type=int, default=0)
a = ap.parse_args()
ext = [int(x) for x in a.shape.split(",")]
prog = hg.build_kernel(hg.KernelSpec("heat", 3, 64, 4, "f32")).with_extents(ext)
plan = hg.Plan(prog)
plan.init_fields()
plan.set_tuning(a.chunks)
plan.run(4)
plan.download(0)
print("ok", plan.kernel_name, ext)
