import os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "oracle"))
import paper_2404_02218_b200 as hg
from oracle import Port
port = Port()

def prog_text(elem, zlo, ylo, nops_variant):
    fb = "[-1,13]x[-2,12]x[-1,17]"
    ft = f"!field<{fb}x{elem}>"
    return f"""builtin.module {{
  func.func @p(%u : {ft}, %gx : {ft}, %gy : {ft}) {{
    %tu = stencil.load %u : {ft} -> !temp<?x{elem}>
    %a1, %a2 = stencil.apply(%a = %tu : !temp<?x{elem}>) -> (!temp<?x{elem}>, !temp<?x{elem}>) {{
      %c = stencil.access %a[0,0,0] : {elem}
      %xp = stencil.access %a[1,0,0] : {elem}
      %yp = stencil.access %a[0,1,0] : {elem}
      %dx = arith.subf %xp, %c : {elem}
      %dy = arith.subf %yp, %c : {elem}
      stencil.return %dx, %dy : {elem}, {elem}
    }}
    stencil.store %a1 to %gx ([{zlo},12]x[{ylo},10]x[0,16]) : !temp<?x{elem}> to {ft}
    stencil.store %a2 to %gy ([{zlo},12]x[{ylo},10]x[0,16]) : !temp<?x{elem}> to {ft}
    func.return
  }}
}}
"""

for elem in ("f64", "f32"):
    for zlo, ylo in ((-1, -1), (0, 0), (-1, 0), (0, -1)):
        prog, _, _ = hg.Program.parse(prog_text(elem, zlo, ylo, 0))
        bad = []
        for rep in range(4):
            plan = hg.Plan(prog); plan.init_fields(); plan.run(1)
            perm, _ = plan.binding(); got = [plan.download(p) for p in perm]
            arrays = port.initial_fields(prog); po = port.run(prog, arrays, 1)
            for i, (a, o) in enumerate(zip(got, [arrays[p] for p in po])):
                m = a != o
                if m.any():
                    bad.append((rep, i, int(m.sum()), np.argwhere(m)[:3].tolist()))
            name = plan.kernel_name
            plan.close()
        print(elem, zlo, ylo, name, bad[:4])
