"""Repeat the multi-apply per-apply tier (HG_NO_FUSE_APPLIES=1) on flux3d and report every
mismatch against the oracle (buffer, count, z planes, values)."""
import os, sys
os.environ["HG_NO_FUSE_APPLIES"] = "1"
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "oracle"))
import paper_2404_02218_b200 as hg
from oracle import Port
from paper_2404_02218_b200.programs.flux3d import xir
port = Port()
T = int(os.environ.get("T", "3"))
shapes = [((12, 10, 21), "f64"), ((7, 9, 8), "f64")]
for shape, elem in shapes:
    prog, _, _ = hg.Program.parse(xir(*shape, elem))
    arrays = port.initial_fields(prog)
    po = port.run(prog, arrays, T)
    want = [arrays[p] for p in po]
    nbad = 0
    for rep in range(int(os.environ.get("REPS", "30"))):
        plan = hg.Plan(prog); plan.init_fields(); plan.run(T)
        perm, _ = plan.binding(); got = [plan.download(p) for p in perm]
        name = plan.kernel_name; plan.close()
        for i, (a, o) in enumerate(zip(got, want)):
            m = a != o
            if m.any():
                nbad += 1
                if nbad <= 4:
                    idx = np.argwhere(m)
                    print(shape, elem, name, "T", T, "rep", rep, "buf", i, int(m.sum()),
                          "zs", sorted(set(idx[:, 0].tolist())), "ys", sorted(set(idx[:, 1].tolist())),
                          "xs", sorted(set(idx[:, 2].tolist())), flush=True)
                    for z, y, x in idx[:3].tolist():
                        print("   ", (z, y, x), repr(a[z, y, x]), repr(o[z, y, x]), flush=True)
    print(shape, elem, name, "T", T, {k: v for k, v in os.environ.items() if k.startswith("HG_")},
          "bad runs", nbad, flush=True)
