"""Piacsek-Williams advection (the PSyclone/MONC PW kernel) authored as a stencil-level module.

BASELINE config 4.  The reference has no PW kernel; this is our
authored `.xir` in the reference's own textual syntax: three fields u, v, w (halo 1) in,
three source terms su, sv, sw out, one fused stencil.apply with three results, diagonal
accesses (so `decompose` rejects it: single-GPU).  Array order is [k][j][i] = [z][y][x]
with x (i) fastest, as the reference lays buffers out (buffer.cpp:65-70).

The z-dependent coefficients of the original (tzc1(k), tzc2(k), tzd1(k), tzd2(k)) are
scalar constants here: the stencil dialect has no 1-D / broadcast operand, and the 1-D
arrays are negligible traffic either way (24 B per point: u, v, w read, su, sv, sw written).

    su = tcx*(u[i-1]*(u+u[i-1]) - u[i+1]*(u+u[i+1]))
    su = su + tcy*(u[j-1]*(v[j-1]+v[j-1,i+1]) - u[j+1]*(v+v[i+1]))
    su = su + tzc1*u[k-1]*(w[k-1]+w[k-1,i+1]) - tzc2*u[k+1]*(w+w[i+1])
    sv, sw: the same pattern (see `statements` below)
"""
from __future__ import annotations

COEFFS = {"tcx": 0.0125, "tcy": 0.0125, "tzc1": 0.02, "tzc2": 0.018, "tzd1": 0.021,
          "tzd2": 0.019}


def statements():
    """(result, terms) where every line is `acc (+|-) coeff*a*(b+c)` in Fortran order."""
    U, V, W = "u", "v", "w"
    return {
        "su": [
            ("tcx", (U, (0, 0, -1)), (U, (0, 0, 0)), (U, (0, 0, -1)),
             (U, (0, 0, 1)), (U, (0, 0, 0)), (U, (0, 0, 1))),
            ("tcy", (U, (0, -1, 0)), (V, (0, -1, 0)), (V, (0, -1, 1)),
             (U, (0, 1, 0)), (V, (0, 0, 0)), (V, (0, 0, 1))),
            (("tzc1", "tzc2"), (U, (-1, 0, 0)), (W, (-1, 0, 0)), (W, (-1, 0, 1)),
             (U, (1, 0, 0)), (W, (0, 0, 0)), (W, (0, 0, 1))),
        ],
        "sv": [
            ("tcx", (V, (0, 0, -1)), (U, (0, 0, -1)), (U, (0, 1, -1)),
             (V, (0, 0, 1)), (U, (0, 0, 0)), (U, (0, 1, 0))),
            ("tcy", (V, (0, -1, 0)), (V, (0, 0, 0)), (V, (0, -1, 0)),
             (V, (0, 1, 0)), (V, (0, 0, 0)), (V, (0, 1, 0))),
            (("tzc1", "tzc2"), (V, (-1, 0, 0)), (W, (-1, 0, 0)), (W, (-1, 1, 0)),
             (V, (1, 0, 0)), (W, (0, 0, 0)), (W, (0, 1, 0))),
        ],
        "sw": [
            ("tcx", (W, (0, 0, -1)), (U, (0, 0, -1)), (U, (1, 0, -1)),
             (W, (0, 0, 1)), (U, (0, 0, 0)), (U, (1, 0, 0))),
            ("tcy", (W, (0, -1, 0)), (V, (0, -1, 0)), (V, (1, -1, 0)),
             (W, (0, 1, 0)), (V, (0, 0, 0)), (V, (1, 0, 0))),
            (("tzd1", "tzd2"), (W, (-1, 0, 0)), (W, (0, 0, 0)), (W, (-1, 0, 0)),
             (W, (1, 0, 0)), (W, (0, 0, 0)), (W, (1, 0, 0))),
        ],
    }


def xir(nz: int, ny: int, nx: int, dtype: str = "f32") -> str:
    """The module text (parsed by the reference's parser, parser.cpp)."""
    ft = f"!field<[-1,{nz + 1}]x[-1,{ny + 1}]x[-1,{nx + 1}]x{dtype}>"
    lines = []
    emit = lines.append
    emit("builtin.module {")
    emit(f"  func.func @pw_advection(%u : {ft}, %v : {ft}, %w : {ft}, %su : {ft}, "
         f"%sv : {ft}, %sw : {ft}) {{")
    for f in "uvw":
        emit(f"    %t{f} = stencil.load %{f} : {ft} -> !temp<?x{dtype}>")
    emit(f"    %r0, %r1, %r2 = stencil.apply(%a = %tu : !temp<?x{dtype}>, %b = %tv : "
         f"!temp<?x{dtype}>, %c = %tw : !temp<?x{dtype}>) -> (!temp<?x{dtype}>, "
         f"!temp<?x{dtype}>, !temp<?x{dtype}>) {{")
    arg = {"u": "%a", "v": "%b", "w": "%c"}
    n = [0]

    def new():
        n[0] += 1
        return f"%x{n[0]}"

    def acc(fa):
        f, (dz, dy, dx) = fa
        nm = new()
        emit(f"      {nm} = stencil.access {arg[f]}[{dz},{dy},{dx}] : {dtype}")
        return nm

    def cst(name):
        nm = new()
        v = COEFFS[name]
        emit(f"      {nm} = arith.constant {v!r} : {dtype}")
        return nm

    def op(kind, a, b):
        nm = new()
        emit(f"      {nm} = arith.{kind} {a}, {b} : {dtype}")
        return nm

    results = []
    for res, lines3 in statements().items():
        val = None
        for t, (coef, a1, b1, c1, a2, b2, c2) in enumerate(lines3):
            if isinstance(coef, tuple):     # acc + c1*a1*(b1+c1) - c2*a2*(b2+c2)
                p1 = op("mulf", op("mulf", cst(coef[0]), acc(a1)), op("addf", acc(b1), acc(c1)))
                p2 = op("mulf", op("mulf", cst(coef[1]), acc(a2)), op("addf", acc(b2), acc(c2)))
                val = op("subf", op("addf", val, p1), p2)
            else:                           # [acc +] coef*(a1*(b1+c1) - a2*(b2+c2))
                d = op("subf", op("mulf", acc(a1), op("addf", acc(b1), acc(c1))),
                       op("mulf", acc(a2), op("addf", acc(b2), acc(c2))))
                term = op("mulf", cst(coef), d)
                val = term if val is None else op("addf", val, term)
        results.append(val)
    emit(f"      stencil.return {', '.join(results)} : {dtype}, {dtype}, {dtype}")
    emit("    }")
    for k, f in enumerate(["su", "sv", "sw"]):
        emit(f"    stencil.store %r{k} to %{f} ([0,{nz}]x[0,{ny}]x[0,{nx}]) : "
             f"!temp<?x{dtype}> to {ft}")
    emit("    func.return")
    emit("  }")
    emit("}")
    return "\n".join(lines) + "\n"
