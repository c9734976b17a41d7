"""One resident 2D heat launch (BASELINE config 1 shape) for ncu: heat2d SDO2 1024^2, 200 steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg  # noqa: E402

prog = hg.build_kernel(hg.KernelSpec("heat", 2, 1024, 2, "f32"))
plan = hg.Plan(prog)
plan.init_fields()
for _ in range(4):
    plan.run(int(os.environ.get("STEPS", "200")))
plan.download(0)
print(plan.kernel_name)
plan.close()
