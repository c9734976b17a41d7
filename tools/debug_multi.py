"""Debug helper: run each random / authored multi-apply module in its own process (JIT multi vs
oracle) and report the first mismatching index per slot."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json
import numpy as np
sys.path.insert(0, %r); sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2404_02218_b200 as hg
from oracle import Port
text = open(sys.argv[1]).read()
prog, _, _ = hg.Program.parse(text)
plan = hg.Plan(prog); plan.init_fields(); plan.run(%d)
perm, _ = plan.binding(); got = [plan.download(p) for p in perm]; name = plan.kernel_name
port = Port(); arrays = port.initial_fields(prog); po = port.run(prog, arrays, %d)
bad = []
for i, (g, o) in enumerate(zip(got, [arrays[p] for p in po])):
    m = ~((g == o) | (np.isnan(g) & np.isnan(o)))
    if m.any():
        idx = np.argwhere(m)
        bad.append((i, int(m.sum()), idx[:3].tolist(), idx[-1].tolist(), list(g.shape)))
print(name, "perm", perm == po, "bad", bad)
'''

if __name__ == "__main__":
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import randprog
    T = 3
    texts = []
    g = json.load(open(os.path.join(REPO, "tests", "golden", "reference_golden.json")))
    texts += [(c["name"], c["text"]) for c in g["authored"] if "applies" in c["program"]]
    ref = None
    try:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        from oracle import Ref
        ref = Ref()
    except Exception as e:
        print("no ref:", e)
    if ref:
        for s in range(100, 130):
            texts.append((f"multi{s}", ref.print(ref.pipeline(ref.parse(randprog.multi_apply(s)), "propagate-bounds"))))
        for s in range(60):
            texts.append((f"single{s}", randprog.single_apply(s)))
    for name, text in texts:
        fn = "/tmp/_m.xir"
        open(fn, "w").write(text)
        r = subprocess.run([sys.executable, "-c", CHILD % (REPO, os.path.join(REPO, "oracle"), os.path.join(REPO, "tests"), T, T), fn],
                           capture_output=True, text=True, timeout=300)
        out = (r.stdout.strip().splitlines() or [""])[-1]
        if r.returncode != 0 or "bad []" not in out:
            print(name, "rc", r.returncode, out, r.stderr.strip().splitlines()[-1:] if r.returncode else "")
    print("done")
