"""Timing of the authored two-stage flux step (multi-apply) per family.
usage: python tools/multi_bench.py [N] [STEPS]"""
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch
sys.path.insert(0, %r)
import paper_2404_02218_b200 as hg
from paper_2404_02218_b200.programs.flux3d import xir
n, T = %d, %d
prog, _, _ = hg.Program.parse(xir(n, n, n))
plan = hg.Plan(prog)
plan.init_fields()
plan.run(3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); plan.run(T); e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
l = plan.launch_count()
print(plan.kernel_name, "%%.1f GPts/s" %% (n ** 3 * T / ms / 1e6), "(8 B/pt ideal -> %%.2f of HBM)" %% (n ** 3 * T / ms / 1e6 * 8 / 6451.8))
'''

if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    for flags in ({"HG_NO_FUSE_APPLIES": "1", "HG_NO_APPLY_JIT": "1"},
                  {"HG_NO_FUSE_APPLIES": "1"}, {}):
        env = dict(os.environ, **flags)
        subprocess.run([sys.executable, "-c", CHILD % (REPO, n, T)], env=env, check=True)
