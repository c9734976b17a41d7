"""Two-stage flux-form diffusion step, authored as a multi-apply stencil module.

A producer apply computes the three face fluxes of u over the core widened by one point
(fx = c*(u - u[i-1]), same along j and k); a consumer apply takes their divergence and updates
u (time slots [[0, 1]]: u_new replaces u next step).  The consumer reads the producer's
temps at +1 offsets -- the "apply consuming apply" form the reference materializes
(stencil_transforms.cpp:334-379, interpreter.cpp:713-758) and `decompose` rejects.  Types carry
explicit bounds, so the module needs no propagate-bounds pass to be read.
"""
from __future__ import annotations


def xir(nz: int, ny: int, nx: int, elem: str = "f32") -> str:
    h = 2
    fb = f"[{-h},{nz + h}]x[{-h},{ny + h}]x[{-h},{nx + h}]"
    ft = f"!field<{fb}x{elem}>"
    tb = f"!temp<[0,{nz + 1}]x[0,{ny + 1}]x[0,{nx + 1}]x{elem}>"
    cb = f"[0,{nz}]x[0,{ny}]x[0,{nx}]"
    ct = f"!temp<{cb}x{elem}>"
    lt = f"!temp<{fb}x{elem}>"
    return f"""builtin.module attributes {{stencil.time_slots = [[0, 1]]}} {{
  func.func @flux(%u : {ft}, %un : {ft}) {{
    %t = stencil.load %u : {ft} -> {lt}
    %fx, %fy, %fz = stencil.apply(%a = %t : {lt}) -> ({tb}, {tb}, {tb}) {{
      %c = stencil.access %a[0,0,0] : {elem}
      %xm = stencil.access %a[0,0,-1] : {elem}
      %ym = stencil.access %a[0,-1,0] : {elem}
      %zm = stencil.access %a[-1,0,0] : {elem}
      %k = arith.constant 0.125 : {elem}
      %dx = arith.subf %c, %xm : {elem}
      %dy = arith.subf %c, %ym : {elem}
      %dz = arith.subf %c, %zm : {elem}
      %gx = arith.mulf %k, %dx : {elem}
      %gy = arith.mulf %k, %dy : {elem}
      %gz = arith.mulf %k, %dz : {elem}
      stencil.return %gx, %gy, %gz : {elem}, {elem}, {elem}
    }}
    %o = stencil.apply(%p = %fx : {tb}, %q = %fy : {tb}, %r = %fz : {tb}, %s = %t : {lt}) -> {ct} {{
      %px = stencil.access %p[0,0,1] : {elem}
      %p0 = stencil.access %p[0,0,0] : {elem}
      %qy = stencil.access %q[0,1,0] : {elem}
      %q0 = stencil.access %q[0,0,0] : {elem}
      %rz = stencil.access %r[1,0,0] : {elem}
      %r0 = stencil.access %r[0,0,0] : {elem}
      %u0 = stencil.access %s[0,0,0] : {elem}
      %ex = arith.subf %px, %p0 : {elem}
      %ey = arith.subf %qy, %q0 : {elem}
      %ez = arith.subf %rz, %r0 : {elem}
      %e1 = arith.addf %ex, %ey : {elem}
      %e2 = arith.addf %e1, %ez : {elem}
      %v = arith.addf %u0, %e2 : {elem}
      stencil.return %v : {elem}
    }}
    stencil.store %o to %un ({cb}) : {ct} to {ft}
    func.return
  }}
}}
"""
