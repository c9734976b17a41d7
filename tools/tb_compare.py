"""A/B timing of the two-step pass (HG_TB=1) against the single-step star on one GPU.
usage: python tools/tb_compare.py ORDER EXTENT [STEPS]"""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2404_02218_b200 as hg
order, n, T = %d, %d, %d
prog = hg.build_kernel(hg.KernelSpec("heat", 3, n, order, "f32"))
plan = hg.Plan(prog)
plan.init_fields()
plan.run(6)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan.run(T); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(plan.kernel_name, "%%.1f GPts/s" %% (n ** 3 * T / ms / 1e6))
'''

if __name__ == "__main__":
    order, n = int(sys.argv[1]), int(sys.argv[2])
    T = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    for tb in ("0", "1"):
        env = dict(os.environ, HG_TB=tb)
        subprocess.run([sys.executable, "-c", CHILD % (REPO, order, n, T)], env=env, check=True)
