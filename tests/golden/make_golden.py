"""Generates tests/golden/*.json from the REAL reference (oracle/_ref/libhalogen_ref.so).

Run in the build container, where /root/reference exists:
    make -C oracle ref && python tests/golden/make_golden.py
Every number in the fixtures comes from the reference's own public API (buildKernel,
initialFields, runSerialStencil, runPipeline("propagate-bounds,decompose ..."), simulate,
initValue, StandardSlicing::exchanges, neighborRank, localInterval, bindingAfter), driven
through oracle/ref_capi.cpp.  Nothing here is computed by our code.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import random
import struct
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
from oracle import Ref  # noqa: E402

from paper_2404_02218_b200 import _capi as capi  # noqa: E402  (descriptor structs only)

# Authored stencil-level modules (our own test inputs in the reference's textual syntax):
# a widened 1-D three-point sum, a 2-D mixed-op stencil with a divide, and a 3-D three-field
# three-result advection-style program with diagonal accesses (generic kernel family).
AUTHORED = {
    "sum3_1d": """builtin.module {
  func.func @sum3(%in : !field<[-1,129]xf32>, %out : !field<[0,128]xf32>) {
    %t = stencil.load %in : !field<[-1,129]xf32> -> !temp<?xf32>
    %o = stencil.apply(%a = %t : !temp<?xf32>) -> !temp<?xf32> {
      %l = stencil.access %a[-1] : f32
      %c = stencil.access %a[0] : f32
      %r = stencil.access %a[1] : f32
      %s0 = arith.addf %l, %c : f32
      %s1 = arith.addf %s0, %r : f32
      stencil.return %s1 : f32
    }
    stencil.store %o to %out ([0,128]) : !temp<?xf32> to !field<[0,128]xf32>
    func.return
  }
}
""",
    "mixed_2d": """builtin.module attributes {stencil.time_slots = [[0, 1]]} {
  func.func @step(%u : !field<[-1,33]x[-2,26]xf32>, %v : !field<[-1,33]x[-2,26]xf32>) {
    %t = stencil.load %u : !field<[-1,33]x[-2,26]xf32> -> !temp<?xf32>
    %o = stencil.apply(%a = %t : !temp<?xf32>) -> !temp<?xf32> {
      %n = stencil.access %a[-1,0] : f32
      %s = stencil.access %a[1,0] : f32
      %w = stencil.access %a[0,-2] : f32
      %e = stencil.access %a[0,1] : f32
      %c = stencil.access %a[0,0] : f32
      %k = arith.constant 3.0 : f32
      %h = arith.constant 0.25 : f32
      %ns = arith.subf %n, %s : f32
      %we = arith.mulf %w, %e : f32
      %q = arith.divf %ns, %k : f32
      %p = arith.addf %q, %we : f32
      %m = arith.mulf %p, %h : f32
      %r = arith.addf %m, %c : f32
      stencil.return %r : f32
    }
    stencil.store %o to %v ([0,32]x[0,24]) : !temp<?xf32> to !field<[-1,33]x[-2,26]xf32>
    func.return
  }
}
""",
    "advect3_3d": """builtin.module {
  func.func @advect(%u : !field<[-1,17]x[-1,13]x[-1,21]xf32>, %v : !field<[-1,17]x[-1,13]x[-1,21]xf32>, %w : !field<[-1,17]x[-1,13]x[-1,21]xf32>, %su : !field<[-1,17]x[-1,13]x[-1,21]xf32>, %sv : !field<[-1,17]x[-1,13]x[-1,21]xf32>, %sw : !field<[-1,17]x[-1,13]x[-1,21]xf32>) {
    %tu = stencil.load %u : !field<[-1,17]x[-1,13]x[-1,21]xf32> -> !temp<?xf32>
    %tv = stencil.load %v : !field<[-1,17]x[-1,13]x[-1,21]xf32> -> !temp<?xf32>
    %tw = stencil.load %w : !field<[-1,17]x[-1,13]x[-1,21]xf32> -> !temp<?xf32>
    %o0, %o1, %o2 = stencil.apply(%a = %tu : !temp<?xf32>, %b = %tv : !temp<?xf32>, %c = %tw : !temp<?xf32>) -> (!temp<?xf32>, !temp<?xf32>, !temp<?xf32>) {
      %half = arith.constant 0.5 : f32
      %u0 = stencil.access %a[0,0,0] : f32
      %up = stencil.access %a[0,0,1] : f32
      %um = stencil.access %a[0,0,-1] : f32
      %vu = stencil.access %b[0,1,-1] : f32
      %wu = stencil.access %c[1,0,-1] : f32
      %d1 = arith.subf %up, %um : f32
      %f1 = arith.mulf %u0, %d1 : f32
      %g1 = arith.mulf %vu, %wu : f32
      %h1 = arith.addf %f1, %g1 : f32
      %r1 = arith.mulf %h1, %half : f32
      %v0 = stencil.access %b[0,0,0] : f32
      %vp = stencil.access %b[0,1,0] : f32
      %vm = stencil.access %b[0,-1,0] : f32
      %uv = stencil.access %a[0,-1,1] : f32
      %d2 = arith.subf %vp, %vm : f32
      %f2 = arith.mulf %v0, %d2 : f32
      %h2 = arith.subf %f2, %uv : f32
      %r2 = arith.mulf %h2, %half : f32
      %w0 = stencil.access %c[0,0,0] : f32
      %wp = stencil.access %c[1,0,0] : f32
      %wm = stencil.access %c[-1,0,0] : f32
      %uw = stencil.access %a[-1,0,1] : f32
      %d3 = arith.subf %wp, %wm : f32
      %f3 = arith.mulf %w0, %d3 : f32
      %x3 = arith.divf %f3, %half : f32
      %r3 = arith.addf %x3, %uw : f32
      stencil.return %r1, %r2, %r3 : f32, f32, f32
    }
    stencil.store %o0 to %su ([0,16]x[0,12]x[0,20]) : !temp<?xf32> to !field<[-1,17]x[-1,13]x[-1,21]xf32>
    stencil.store %o1 to %sv ([0,16]x[0,12]x[0,20]) : !temp<?xf32> to !field<[-1,17]x[-1,13]x[-1,21]xf32>
    stencil.store %o2 to %sw ([0,16]x[0,12]x[0,20]) : !temp<?xf32> to !field<[-1,17]x[-1,13]x[-1,21]xf32>
    func.return
  }
}
""",
}

# Multi-apply modules (one apply consuming another's result temp, several results, and
# independent applies in one step) -- the stencil-level form the reference interprets
# apply by apply (interpreter.cpp stencil.apply / stencil.store handlers).
AUTHORED["flux2_2d"] = """builtin.module attributes {stencil.time_slots = [[0, 1]]} {
  func.func @flux(%u : !field<[-2,34]x[-2,26]xf32>, %v : !field<[-2,34]x[-2,26]xf32>) {
    %t = stencil.load %u : !field<[-2,34]x[-2,26]xf32> -> !temp<?xf32>
    %f = stencil.apply(%a = %t : !temp<?xf32>) -> !temp<?xf32> {
      %c = stencil.access %a[0,0] : f32
      %e = stencil.access %a[1,0] : f32
      %d = arith.subf %e, %c : f32
      %k = arith.constant 0.3 : f32
      %r = arith.mulf %d, %k : f32
      stencil.return %r : f32
    }
    %o = stencil.apply(%b = %f : !temp<?xf32>, %x = %t : !temp<?xf32>) -> !temp<?xf32> {
      %fp = stencil.access %b[0,0] : f32
      %fm = stencil.access %b[-1,0] : f32
      %df = arith.subf %fp, %fm : f32
      %xc = stencil.access %x[0,1] : f32
      %xs = arith.addf %xc, %df : f32
      stencil.return %xs : f32
    }
    stencil.store %o to %v ([0,32]x[0,24]) : !temp<?xf32> to !field<[-2,34]x[-2,26]xf32>
    func.return
  }
}
"""
AUTHORED["chain3_3d_f64"] = """builtin.module attributes {stencil.time_slots = [[0, 2]]} {
  func.func @chain(%u : !field<[-1,13]x[-2,12]x[-1,17]xf64>, %w : !field<[-1,13]x[-2,12]x[-1,17]xf64>, %un : !field<[-1,13]x[-2,12]x[-1,17]xf64>, %s : !field<[-1,13]x[-2,12]x[-1,17]xf64>) {
    %tu = stencil.load %u : !field<[-1,13]x[-2,12]x[-1,17]xf64> -> !temp<?xf64>
    %tw = stencil.load %w : !field<[-1,13]x[-2,12]x[-1,17]xf64> -> !temp<?xf64>
    %gx, %gy = stencil.apply(%a = %tu : !temp<?xf64>) -> (!temp<?xf64>, !temp<?xf64>) {
      %c = stencil.access %a[0,0,0] : f64
      %xp = stencil.access %a[1,0,0] : f64
      %yp = stencil.access %a[0,1,0] : f64
      %dx = arith.subf %xp, %c : f64
      %dy = arith.subf %yp, %c : f64
      stencil.return %dx, %dy : f64, f64
    }
    %m = stencil.apply(%p = %gx : !temp<?xf64>, %q = %gy : !temp<?xf64>, %r = %tw : !temp<?xf64>) -> !temp<?xf64> {
      %px = stencil.access %p[0,0,0] : f64
      %pm = stencil.access %p[-1,0,0] : f64
      %qy = stencil.access %q[0,0,0] : f64
      %qm = stencil.access %q[0,-1,0] : f64
      %rz = stencil.access %r[0,0,1] : f64
      %lx = arith.subf %px, %pm : f64
      %ly = arith.subf %qy, %qm : f64
      %l = arith.addf %lx, %ly : f64
      %h = arith.constant 0.125 : f64
      %hl = arith.mulf %h, %l : f64
      %o1 = arith.addf %rz, %hl : f64
      stencil.return %o1 : f64
    }
    %k = stencil.apply(%z = %tw : !temp<?xf64>) -> !temp<?xf64> {
      %zc = stencil.access %z[0,0,0] : f64
      %zm = stencil.access %z[0,-2,-1] : f64
      %zd = arith.divf %zm, %zc : f64
      stencil.return %zd : f64
    }
    stencil.store %m to %un ([0,12]x[0,10]x[0,16]) : !temp<?xf64> to !field<[-1,13]x[-2,12]x[-1,17]xf64>
    stencil.store %k to %s ([0,12]x[0,10]x[0,16]) : !temp<?xf64> to !field<[-1,13]x[-2,12]x[-1,17]xf64>
    func.return
  }
}
"""
AUTHORED["indep2_2d"] = """builtin.module {
  func.func @two(%a : !field<[-1,41]x[-1,9]xf32>, %b : !field<[-1,41]x[-1,9]xf32>, %c : !field<[-1,41]x[-1,9]xf32>, %d : !field<[-1,41]x[-1,9]xf32>) {
    %ta = stencil.load %a : !field<[-1,41]x[-1,9]xf32> -> !temp<?xf32>
    %tb = stencil.load %b : !field<[-1,41]x[-1,9]xf32> -> !temp<?xf32>
    %o1 = stencil.apply(%x = %ta : !temp<?xf32>) -> !temp<?xf32> {
      %x0 = stencil.access %x[-1,1] : f32
      %x1 = stencil.access %x[1,-1] : f32
      %x2 = arith.addf %x0, %x1 : f32
      stencil.return %x2 : f32
    }
    %o2 = stencil.apply(%y = %tb : !temp<?xf32>, %yy = %ta : !temp<?xf32>) -> !temp<?xf32> {
      %y0 = stencil.access %y[0,0] : f32
      %y1 = stencil.access %yy[0,1] : f32
      %y2 = arith.mulf %y0, %y1 : f32
      stencil.return %y2 : f32
    }
    stencil.store %o1 to %c ([0,40]x[0,8]) : !temp<?xf32> to !field<[-1,41]x[-1,9]xf32>
    stencil.store %o2 to %d ([0,40]x[0,8]) : !temp<?xf32> to !field<[-1,41]x[-1,9]xf32>
    func.return
  }
}
"""

# Decomposable multi-apply modules (independent applies, face footprints, symmetric halos):
# decompose inserts a swap before every load (dmp_transforms.cpp:276-300).
DECOMP_AUTHORED = {
    "indep2f_2d": ("""builtin.module attributes {stencil.time_slots = [[0, 2], [1, 3]]} {
  func.func @two(%a : !field<[-1,41]x[-1,9]xf32>, %b : !field<[-1,41]x[-1,9]xf32>, %c : !field<[-1,41]x[-1,9]xf32>, %d : !field<[-1,41]x[-1,9]xf32>) {
    %ta = stencil.load %a : !field<[-1,41]x[-1,9]xf32> -> !temp<?xf32>
    %tb = stencil.load %b : !field<[-1,41]x[-1,9]xf32> -> !temp<?xf32>
    %o1 = stencil.apply(%x = %ta : !temp<?xf32>) -> !temp<?xf32> {
      %x0 = stencil.access %x[-1,0] : f32
      %x1 = stencil.access %x[0,-1] : f32
      %x2 = arith.addf %x0, %x1 : f32
      %x3 = arith.constant 0.5 : f32
      %x4 = arith.mulf %x2, %x3 : f32
      stencil.return %x4 : f32
    }
    %o2 = stencil.apply(%y = %tb : !temp<?xf32>, %yy = %ta : !temp<?xf32>) -> !temp<?xf32> {
      %y0 = stencil.access %y[1,0] : f32
      %y1 = stencil.access %yy[0,1] : f32
      %y2 = arith.subf %y0, %y1 : f32
      stencil.return %y2 : f32
    }
    stencil.store %o1 to %c ([0,40]x[0,8]) : !temp<?xf32> to !field<[-1,41]x[-1,9]xf32>
    stencil.store %o2 to %d ([0,40]x[0,8]) : !temp<?xf32> to !field<[-1,41]x[-1,9]xf32>
    func.return
  }
}
""", [2, 2], 3),
    "twin3_3d_f64": ("""builtin.module attributes {stencil.time_slots = [[0, 2], [1, 3]]} {
  func.func @twin(%u : !field<[-2,18]x[-1,13]x[-1,17]xf64>, %v : !field<[-2,18]x[-1,13]x[-1,17]xf64>, %un : !field<[-2,18]x[-1,13]x[-1,17]xf64>, %vn : !field<[-2,18]x[-1,13]x[-1,17]xf64>) {
    %tv = stencil.load %v : !field<[-2,18]x[-1,13]x[-1,17]xf64> -> !temp<?xf64>
    %tu = stencil.load %u : !field<[-2,18]x[-1,13]x[-1,17]xf64> -> !temp<?xf64>
    %ou = stencil.apply(%a = %tu : !temp<?xf64>) -> !temp<?xf64> {
      %c = stencil.access %a[0,0,0] : f64
      %zp = stencil.access %a[2,0,0] : f64
      %zm = stencil.access %a[-2,0,0] : f64
      %yp = stencil.access %a[0,1,0] : f64
      %xm = stencil.access %a[0,0,-1] : f64
      %s1 = arith.addf %zp, %zm : f64
      %s2 = arith.addf %yp, %xm : f64
      %s3 = arith.addf %s1, %s2 : f64
      %k = arith.constant 0.2 : f64
      %s4 = arith.mulf %k, %s3 : f64
      %s5 = arith.subf %s4, %c : f64
      stencil.return %s5 : f64
    }
    %ov = stencil.apply(%p = %tv : !temp<?xf64>, %q = %tu : !temp<?xf64>) -> !temp<?xf64> {
      %pc = stencil.access %p[0,0,1] : f64
      %py = stencil.access %p[0,-1,0] : f64
      %qz = stencil.access %q[1,0,0] : f64
      %m = arith.mulf %pc, %qz : f64
      %n = arith.divf %m, %py : f64
      stencil.return %n : f64
    }
    stencil.store %ou to %un ([0,16]x[0,12]x[0,16]) : !temp<?xf64> to !field<[-2,18]x[-1,13]x[-1,17]xf64>
    stencil.store %ov to %vn ([0,16]x[0,12]x[0,16]) : !temp<?xf64> to !field<[-2,18]x[-1,13]x[-1,17]xf64>
    func.return
  }
}
""", [2, 2, 2], 3),
}

sys.path.insert(0, REPO)
from paper_2404_02218_b200.programs.pw_advection import xir as pw_xir  # noqa: E402

AUTHORED["pw_advection_16x24x40"] = pw_xir(16, 24, 40)
AUTHORED["pw_advection_f64_9x10x11"] = pw_xir(9, 10, 11, "f64")
from paper_2404_02218_b200.programs.flux3d import xir as flux_xir  # noqa: E402

AUTHORED["flux3d_12x10x21"] = flux_xir(12, 10, 21)
AUTHORED["flux3d_f64_7x9x8"] = flux_xir(7, 9, 8, "f64")

SERIAL = [  # (kind, rank, extent, order, f32, T)
    ("heat", 1, 16, 2, 1, 5), ("heat", 1, 128, 8, 0, 7),
    ("heat", 2, 16, 2, 1, 5), ("heat", 2, 16, 2, 0, 5), ("heat", 2, 12, 4, 1, 3),
    ("heat", 2, 40, 8, 1, 4), ("heat", 2, 100, 2, 1, 6), ("heat", 2, 257, 4, 1, 3),
    ("heat", 3, 8, 4, 1, 3), ("heat", 3, 8, 4, 0, 3), ("heat", 3, 12, 8, 1, 2),
    ("heat", 3, 20, 2, 1, 4), ("heat", 3, 33, 4, 1, 3), ("heat", 3, 64, 4, 1, 4),
    ("heat", 3, 24, 8, 0, 2),
    ("wave", 1, 16, 4, 1, 4), ("wave", 2, 16, 8, 1, 3), ("wave", 2, 70, 4, 0, 3),
    ("wave", 3, 10, 4, 1, 3), ("wave", 3, 12, 8, 1, 2), ("wave", 3, 48, 8, 1, 3),
    ("wave", 3, 17, 2, 0, 4), ("wave", 3, 40, 8, 1, 5),
    ("copy", 2, 8, 2, 1, 2), ("copy", 3, 9, 2, 0, 3),
    ("heat", 2, 1024, 2, 1, 0), ("heat", 2, 1024, 2, 1, 1),
]
CONFIG1 = ("heat", 2, 1024, 2, 1, 100)   # BASELINE config 1, the minimum slice

DECOMP = [  # (kind, rank, extent, order, f32, grid, T)
    ("heat", 2, 12, 2, 1, [2, 2], 3), ("wave", 1, 16, 4, 1, [4], 4),
    ("copy", 2, 8, 2, 1, [2, 1], 2), ("heat", 2, 64, 2, 1, [2, 4], 2),
    ("heat", 3, 16, 4, 1, [2, 2, 2], 3), ("wave", 3, 16, 8, 1, [2, 2, 2], 3),
    ("heat", 3, 32, 4, 1, [4, 1, 1], 2), ("heat", 3, 24, 4, 0, [1, 2, 3], 2),
    ("wave", 3, 24, 4, 1, [2, 1, 2], 4), ("heat", 2, 12, 2, 0, [2, 2], 3),
]


def prog_json(prog, ops):
    r = prog.rank
    if prog.napplies > 0:
        aps = prog.applies
        return {
            "rank": r, "dtype": prog.dtype, "nfields": prog.nfields,
            "fields": [[list(prog.fields[i].lb[:r]), list(prog.fields[i].ub[:r])]
                       for i in range(prog.nfields)],
            "ops": [[o.code, o.a, o.b, o.operand, list(o.off[:r]), "%016x" % o.bits]
                    for o in ops[:prog.nops]],
            "applies": [{"operands": list(aps[a].operand[:aps[a].noperands]),
                         "op_begin": aps[a].op_begin, "nops": aps[a].nops,
                         "result_op": list(aps[a].result_op[:aps[a].nresults]),
                         "result_temp": list(aps[a].result_temp[:aps[a].nresults]),
                         "domain": [list(aps[a].domain.lb[:r]), list(aps[a].domain.ub[:r])]}
                        for a in range(prog.napplies)],
            "loads": list(prog.operand_field[:prog.noperands]),
            "ntemps": prog.ntemps,
            "mstores": [[prog.mstore_temp[k], prog.mstore_field[k],
                         list(prog.mstore[k].lb[:r]), list(prog.mstore[k].ub[:r])]
                        for k in range(prog.nstores)],
            "groups": _groups(prog),
        }
    return {
        "rank": r, "dtype": prog.dtype, "nfields": prog.nfields,
        "fields": [[list(prog.fields[i].lb[:r]), list(prog.fields[i].ub[:r])]
                   for i in range(prog.nfields)],
        "operand_field": list(prog.operand_field[:prog.noperands]),
        "ops": [[o.code, o.a, o.b, o.operand, list(o.off[:r]), "%016x" % o.bits]
                for o in ops[:prog.nops]],
        "result_op": list(prog.result_op[:prog.nresults]),
        "store_field": list(prog.store_field[:prog.nresults]),
        "store": [[list(prog.store[k].lb[:r]), list(prog.store[k].ub[:r])]
                  for k in range(prog.nresults)],
        "groups": _groups(prog),
    }


def _groups(prog):
    out, at = [], 0
    for g in range(prog.ngroups):
        out.append(list(prog.groups[at:at + prog.group_len[g]]))
        at += prog.group_len[g]
    return out


def decomp_json(dc):
    n = dc.ndim
    return {"grid": list(dc.grid[:n]), "core": list(dc.core[:n]),
            "swaps": [{"field": s.field,
                       "ex": [[list(e.at[:n]), list(e.size[:n]), list(e.offset[:n]),
                               list(e.to[:n])] for e in s.ex[:s.nexchanges]]}
                      for s in dc.swaps[:dc.nswaps]]}


def fps(ref, bufs):
    return ["%016x" % ref.L.hr_fingerprint(bufs, i) for i in range(ref.L.hr_bufs_count(bufs))]


def main():
    ref = Ref()
    L = ref.L
    out = {"generator": "tests/golden/make_golden.py via oracle/_ref/libhalogen_ref.so "
                        "(reference core compiled from /root/reference/proj/core)"}

    # initValue (buffer.cpp:142-156)
    rng = random.Random(20261018)
    coords = [(0, [0, 0]), (1, [0, 0]), (0, [-1, -1]), (1, [1023, 1024]), (0, [0, 0, 0]),
              (1, [-2, -2, -2]), (0, [511, 511, 511]), (2, [-4, 0, 1027]), (0, [5]),
              (3, [-9, 7])]
    for _ in range(40):
        r = rng.randint(1, 3)
        coords.append((rng.randint(0, 5), [rng.randint(-5000, 5000) for _ in range(r)]))
    iv = []
    for f, c in coords:
        v = L.hr_init_value(f, len(c), (C.c_longlong * len(c))(*c))
        iv.append({"field": f, "coord": c, "f64": struct.pack("<d", v).hex(),
                   "f32": struct.pack("<f", v).hex()})
    out["init_values"] = iv

    # programs + serial runs
    serial = []
    for kind, rank, ext, order, f32, T in SERIAL + [CONFIG1]:
        t0 = time.time()
        mod = ref.build(kind, rank, ext, order, bool(f32))
        prog, ops, _ = ref.export_program(mod)
        init = L.hr_initial_fields(mod)
        work = L.hr_bufs_clone(init)
        fin = L.hr_run_serial(mod, work, T)
        if not fin:
            raise RuntimeError(ref.err())
        serial.append({"spec": [kind, rank, ext, order, f32], "T": T,
                       "program": prog_json(prog, ops),
                       "text": ref.print(mod) if ext <= 40 else None,
                       "init_fp": fps(ref, init), "final_fp": fps(ref, fin),
                       "seconds": time.time() - t0})
        for b in (init, work, fin):
            L.hr_bufs_free(b)
        L.hr_module_free(mod)
        print("serial", kind, rank, ext, order, f32, T, "%.2fs" % (time.time() - t0), flush=True)
    out["serial"] = serial

    # authored modules
    auth = []
    for name, text in AUTHORED.items():
        mod = ref.pipeline(ref.parse(text), "propagate-bounds")
        prog, ops, _ = ref.export_program(mod)
        init = L.hr_initial_fields(mod)
        work = L.hr_bufs_clone(init)
        T = 3 if prog.ngroups else 1
        fin = L.hr_run_serial(mod, work, T)
        if not fin:
            raise RuntimeError(ref.err())
        auth.append({"name": name, "T": T, "program": prog_json(prog, ops),
                     "text": ref.print(mod),
                     "init_fp": fps(ref, init), "final_fp": fps(ref, fin)})
        if name == "pw_advection_16x24x40":  # the authored config-4 program, as data
            with open(os.path.join(REPO, "paper_2404_02218_b200", "programs",
                                   "pw_advection.json"), "w") as f:
                json.dump({"generator": "reference parser + propagate-bounds on "
                                        "programs/pw_advection.py:xir(16,24,40)",
                           "program": prog_json(prog, ops)}, f, indent=1)
        print("authored", name, flush=True)
    out["authored"] = auth

    # decompose + simulate (dmp level, RankHooks::swap)
    dec = []
    for kind, rank, ext, order, f32, grid, T in DECOMP:
        mod = ref.build(kind, rank, ext, order, bool(f32))
        gs = "x".join(str(g) for g in grid)
        dmod = ref.pipeline(mod, "propagate-bounds,decompose grid=" + gs)
        lprog, lops, dc = ref.export_program(dmod)
        init = L.hr_initial_fields(mod)
        res = L.hr_simulate(dmod, init, T, 0)
        if not res:
            raise RuntimeError(ref.err())
        ser = L.hr_run_serial(mod, L.hr_bufs_clone(init), T)
        # also the fully lowered mpi level, as `halogen bench --grid` times it
        mmod = ref.pipeline(mod, "propagate-bounds,decompose grid=" + gs + ",lower-dmp-to-mpi")
        mres = L.hr_simulate(mmod, init, T, 0)
        if not mres:
            raise RuntimeError(ref.err())
        dec.append({"spec": [kind, rank, ext, order, f32], "grid": grid, "T": T,
                    "local_program": prog_json(lprog, lops), "decomp": decomp_json(dc),
                    "text": ref.print(dmod),
                    "sim_fp": fps(ref, res), "mpi_sim_fp": fps(ref, mres),
                    "serial_fp": fps(ref, ser)})
        print("decomp", kind, rank, ext, order, grid, T, flush=True)
    out["decomposed"] = dec

    # decomposed multi-apply modules (authored), same record shape + the global program
    dau = []
    for name, (text, grid, T) in DECOMP_AUTHORED.items():
        mod = ref.pipeline(ref.parse(text), "propagate-bounds")
        gprog, gops, _ = ref.export_program(mod)
        gs = "x".join(str(g) for g in grid)
        dmod = ref.pipeline(mod, "propagate-bounds,decompose grid=" + gs)
        lprog, lops, dc = ref.export_program(dmod)
        init = L.hr_initial_fields(mod)
        res = L.hr_simulate(dmod, init, T, 0)
        if not res:
            raise RuntimeError(ref.err())
        ser = L.hr_run_serial(mod, L.hr_bufs_clone(init), T)
        mmod = ref.pipeline(mod, "propagate-bounds,decompose grid=" + gs + ",lower-dmp-to-mpi")
        mres = L.hr_simulate(mmod, init, T, 0)
        if not mres:
            raise RuntimeError(ref.err())
        dau.append({"name": name, "grid": grid, "T": T, "program": prog_json(gprog, gops),
                    "local_program": prog_json(lprog, lops), "decomp": decomp_json(dc),
                    "text": ref.print(dmod), "global_text": ref.print(mod),
                    "init_fp": fps(ref, init), "sim_fp": fps(ref, res),
                    "mpi_sim_fp": fps(ref, mres), "serial_fp": fps(ref, ser)})
        print("decomp authored", name, grid, T, flush=True)
    out["decomposed_authored"] = dau

    # dmp arithmetic (dmp_ops.cpp:21-115)
    dmp = {"exchanges": [], "neighbors": [], "slicing": [], "coords": []}
    LL = C.c_longlong
    a = lambda v: (LL * len(v))(*v)  # noqa: E731
    cases = [([100, 100], [4, 4], [4, 4], None, None), ([8, 8], [0, 2], [0, 2], None, None),
             ([8, 8], [1, 1], [1, 1], [2, 2], [0, 0]), ([8, 8], [1, 1], [1, 1], [3, 3], [1, 1])]
    rng = random.Random(20260816)
    for _ in range(60):
        r = rng.randint(1, 3)
        grid = [rng.randint(1, 4) for _ in range(r)]
        halo = [rng.randint(0, 3) for _ in range(r)]
        core = [max(h, 1) + rng.randint(0, 9) for h in halo]
        coord = [rng.randint(0, g - 1) for g in grid]
        cases.append((core, halo, halo, grid, coord) if rng.random() < 0.7 else
                     (core, halo, halo, None, None))
    for core, lo, hi, grid, coord in cases:
        n = len(core)
        buf = (LL * (24 * n))()
        k = L.hr_exchanges(n, a(core), a(lo), a(hi), a(grid) if grid else None,
                           a(coord) if coord else None, buf, 6)
        decl = [[list(buf[j * 4 * n + q * n: j * 4 * n + (q + 1) * n]) for q in range(4)]
                for j in range(k)]
        dmp["exchanges"].append({"core": core, "below": lo, "above": hi, "grid": grid,
                                 "coord": coord, "decls": decl})
    for grid in ([2, 4, 4], [4], [3, 4], [2, 3, 2], [5]):
        n = len(grid)
        total = 1
        for g in grid:
            total *= g
        for r in range(total):
            c = (LL * n)()
            L.hr_coord_from_rank(n, r, a(grid), c)
            dmp["coords"].append({"grid": grid, "rank": r, "coord": list(c)})
            for d in range(n):
                for s in (-1, 1):
                    dirv = [0] * n
                    dirv[d] = s
                    dmp["neighbors"].append({"grid": grid, "rank": r, "dir": dirv,
                                             "nbr": L.hr_neighbor_rank(n, r, a(dirv), a(grid))})
    rng = random.Random(7)
    for _ in range(200):
        parts = rng.randint(1, 8)
        ext = parts + rng.randint(0, 199)
        for p in range(parts):
            lb, ub = LL(), LL()
            L.hr_local_interval(ext, parts, p, C.byref(lb), C.byref(ub))
            dmp["slicing"].append([ext, parts, p, lb.value, ub.value])
    out["dmp"] = dmp

    # bindingAfter
    ba = []
    for groups, nargs in (([[0, 1]], 2), ([[0, 1, 2]], 3), ([[0, 1]], 3), ([[0, 2], [1, 3, 4]], 5)):
        for steps in (0, 1, 2, 3, 5, 16, 17):
            gl = (C.c_int * len(groups))(*[len(g) for g in groups])
            flat = [i for g in groups for i in g]
            gg = (C.c_int * len(flat))(*flat)
            o = (C.c_int * nargs)()
            L.hr_binding_after(len(groups), gl, gg, nargs, steps, o)
            ba.append({"groups": groups, "nargs": nargs, "steps": steps, "perm": list(o)})
    out["binding_after"] = ba

    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", os.path.join(HERE, "reference_golden.json"))


if __name__ == "__main__":
    main()
