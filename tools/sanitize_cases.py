"""Small cases for compute-sanitizer (tools/runs/gpu_r2_sanitize.sh): every kernel family once,
checked against the oracle so a sanitizer run is also a parity run."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))

import numpy as np  # noqa: E402

import paper_2404_02218_b200 as hg  # noqa: E402
from oracle import Port  # noqa: E402


def check(prog, T, label):
    port = Port()
    arrays = port.initial_fields(prog)
    plan = hg.Plan(prog)
    plan.init_fields()
    plan.run(T)
    perm, _ = plan.binding()
    got = [plan.download(p) for p in perm]
    name = plan.kernel_name
    plan.close()
    perm_o = port.run(prog, arrays, T)
    ok = perm == perm_o and all(np.array_equal(g.view(np.uint8), arrays[p].view(np.uint8))
                                for g, p in zip(got, perm_o))
    print(f"{label}: {name} {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


ok = True
ok &= check(hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents([70, 30, 200]), 3,
            "heat3d so4 (3 chunks, ragged)")
ok &= check(hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents([40, 780, 800]),
            2, "heat3d so4 wide tile")
ok &= check(hg.build_kernel(hg.KernelSpec("wave", 3, 8, 8, "f32")).with_extents([150, 30, 70]), 3,
            "wave3d so8 (2 chunks)")
ok &= check(hg.build_kernel(hg.KernelSpec("heat", 2, 256, 2, "f32")), 5, "heat2d resident")
ok &= check(hg.build_kernel(hg.KernelSpec("heat", 3, 40, 4, "f64")), 2, "heat3d f64")
ok &= check(hg.Program.pw_advection(20, 40, 72), 2, "pw advection (generated)")
from paper_2404_02218_b200.programs.flux3d import xir  # noqa: E402
ok &= check(hg.Program.parse(xir(20, 18, 37))[0], 2, "flux3d multi-apply (fused)")
sys.exit(0 if ok else 1)
