import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import numpy as np
import paper_2404_02218_b200 as hg
from oracle import Port
port = Port()
for spec, grid, T, devs in [(("wave", 3, 24, 8), [3, 1, 1], 4, [0, 1, 0]), (("wave", 3, 24, 8), [3, 1, 1], 4, [0, 0, 0]),
                            (("heat", 3, 24, 4), [3, 1, 1], 4, [0, 1, 0]), (("wave", 3, 24, 8), [3, 1, 1], 1, [0, 1, 0]),
                            (("wave", 3, 24, 8), [2, 1, 1], 3, [0, 1]), (("heat", 2, 24, 2), [2, 2], 3, [0, 1, 0, 1])]:
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    init = hg.initial_fields(prog)
    out = hg.simulate(prog, grid, init, T, devices=devs)
    arrays = [b.data.copy() for b in init]
    perm = port.run(prog, arrays, T)
    bad = []
    for i, (b, p) in enumerate(zip(out, perm)):
        d = np.argwhere(b.data.view(np.uint32) != arrays[p].view(np.uint32))
        if len(d):
            bad.append((i, len(d), d[:3].tolist()))
    print(spec, grid, T, devs, "OK" if not bad else bad, flush=True)
