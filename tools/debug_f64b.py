import os, sys
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "oracle"))
import paper_2404_02218_b200 as hg
from oracle import Port
port = Port()

def cons(elem, variant):
    fb = "[-1,13]x[-2,12]x[-1,17]"
    ft = f"!field<{fb}x{elem}>"
    acc = {"full": ("[0,0,0]", "[-1,0,0]", "[0,0,0]", "[0,-1,0]", "[0,0,1]"),
           "noz": ("[0,0,0]", "[0,0,0]", "[0,0,0]", "[0,-1,0]", "[0,0,1]"),
           "noy": ("[0,0,0]", "[-1,0,0]", "[0,0,0]", "[0,0,0]", "[0,0,1]"),
           "nox": ("[0,0,0]", "[-1,0,0]", "[0,0,0]", "[0,-1,0]", "[0,0,0]")}[variant]
    return f"""builtin.module {{
  func.func @c(%gx : {ft}, %gy : {ft}, %w : {ft}, %un : {ft}) {{
    %tx = stencil.load %gx : {ft} -> !temp<?x{elem}>
    %ty = stencil.load %gy : {ft} -> !temp<?x{elem}>
    %tw = stencil.load %w : {ft} -> !temp<?x{elem}>
    %m = stencil.apply(%p = %tx : !temp<?x{elem}>, %q = %ty : !temp<?x{elem}>, %r = %tw : !temp<?x{elem}>) -> !temp<?x{elem}> {{
      %18 = stencil.access %p{acc[0]} : {elem}
      %19 = stencil.access %p{acc[1]} : {elem}
      %20 = stencil.access %q{acc[2]} : {elem}
      %21 = stencil.access %q{acc[3]} : {elem}
      %22 = stencil.access %r{acc[4]} : {elem}
      %23 = arith.subf %18, %19 : {elem}
      %24 = arith.subf %20, %21 : {elem}
      %25 = arith.addf %23, %24 : {elem}
      %26 = arith.constant 0.125 : {elem}
      %27 = arith.mulf %26, %25 : {elem}
      %28 = arith.addf %22, %27 : {elem}
      stencil.return %28 : {elem}
    }}
    stencil.store %m to %un ([0,12]x[0,10]x[0,16]) : !temp<?x{elem}> to {ft}
    func.return
  }}
}}
"""

for elem in ("f64", "f32"):
    for v in ("full", "noz", "noy", "nox"):
        prog, _, _ = hg.Program.parse(cons(elem, v))
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
        print(elem, v, name, bad[:4])
