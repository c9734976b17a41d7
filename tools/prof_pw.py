"""One PW-advection plan (BASELINE config 4 shape, 128 x 512 x 512, x fastest) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg  # noqa: E402

prog = hg.Program.pw_advection(128, 512, 512)
plan = hg.Plan(prog)
plan.init_fields()
plan.run(int(os.environ.get("STEPS", "4")))
plan.download(0)
print("ok", plan.kernel_name)
plan.close()
