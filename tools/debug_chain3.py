import json, os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "oracle"))
import paper_2404_02218_b200 as hg
from oracle import Port
g = json.load(open(os.path.join(REPO, "tests", "golden", "reference_golden.json")))
text = [c["text"] for c in g["authored"] if c["name"] == "chain3_3d_f64"][0]
port = Port()
for variant in ("f64", "f32"):
    t = text if variant == "f64" else text.replace("f64", "f32")
    prog, _, _ = hg.Program.parse(t)
    for T in (1, 1, 1, 2):
        plan = hg.Plan(prog); plan.init_fields(); plan.run(T)
        perm, _ = plan.binding(); got = [plan.download(p) for p in perm]
        arrays = port.initial_fields(prog); po = port.run(prog, arrays, T)
        res = []
        for i, (a, o) in enumerate(zip(got, [arrays[p] for p in po])):
            m = a != o
            if m.any():
                idx = np.argwhere(m)
                res.append((i, int(m.sum()), idx[:4].tolist()))
        print(variant, "T", T, plan.kernel_name, res)
        plan.close()
