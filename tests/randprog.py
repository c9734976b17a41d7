"""Random stencil-level modules in the reference's textual syntax (printer.cpp / parser.cpp),
for fuzzing the device families against the oracle and the oracle against the reference.

Single-apply modules: 1-3 loaded fields, 1-3 results stored into their own fields, accesses
anywhere inside the field halo (diagonals included), constants, add/sub/mul/div.  Multi-apply
modules: a producer apply (one or two results) over the domain widened by 1, consumed with
offsets in [-1, 1] by a second apply that also reads a field, plus an independent third apply.
"""
import random
import struct


def _f32_literal(rng):
    # a decimal literal whose f32 parse is exact enough to be interesting but never inf/nan
    v = rng.choice([0.5, 0.25, 1.5, 2.0, 0.1, 0.3, 1.0 / 3.0, -0.75, 3.0, 0.01, 1e-3, 7.25])
    return repr(float(struct.unpack("<f", struct.pack("<f", v))[0])) if rng.random() < 0.5 \
        else repr(v)


def _region(rng, names, noperands, r, max_off, nops, results, prefix, elem):
    """Body lines of one apply region; returns (lines, names of the returned values)."""
    lines, vals = [], []
    k = 0

    def fresh():
        nonlocal k
        k += 1
        return f"%{prefix}{k}"
    # at least one access per operand so every operand is used
    for o in range(noperands):
        v = fresh()
        off = [rng.randint(-max_off[o], max_off[o]) for _ in range(r)]
        lines.append(f"      {v} = stencil.access {names[o]}[{','.join(map(str, off))}] : {elem}")
        vals.append(v)
    for _ in range(nops):
        c = rng.random()
        v = fresh()
        if c < 0.3:
            o = rng.randrange(noperands)
            off = [rng.randint(-max_off[o], max_off[o]) for _ in range(r)]
            lines.append(f"      {v} = stencil.access {names[o]}[{','.join(map(str, off))}] : "
                         f"{elem}")
        elif c < 0.42:
            lines.append(f"      {v} = arith.constant {_f32_literal(rng)} : {elem}")
        else:
            op = rng.choice(["addf", "addf", "subf", "mulf", "mulf", "divf"])
            a, b = rng.choice(vals), rng.choice(vals)
            if op in ("subf", "divf") and len(vals) > 1:
                while b == a:  # x-x and x/x invite 0/0 -> NaN, whose payload IEEE leaves open
                    b = rng.choice(vals)
            lines.append(f"      {v} = arith.{op} {a}, {b} : {elem}")
        vals.append(v)
    ret = vals[-results:]
    lines.append(f"      stencil.return {', '.join(ret)} : {', '.join([elem] * results)}")
    return lines


def _btxt(lb, ub):
    return "x".join(f"[{a},{b}]" for a, b in zip(lb, ub))


def single_apply(seed: int):
    rng = random.Random(seed)
    r = rng.choice([2, 3])
    elem = rng.choice(["f32", "f32", "f64"])
    n = [rng.randint(5, 14) for _ in range(r)]
    h = rng.randint(1, 3)
    nin, nout = rng.randint(1, 3), rng.randint(1, 3)
    fb = _btxt([-h] * r, [x + h for x in n])
    ftype = f"!field<{fb}x{elem}>"
    args = [f"%in{i} : {ftype}" for i in range(nin)] + [f"%out{i} : {ftype}" for i in range(nout)]
    # time slots: output i replaces input i next step (ping-pong groups, kernels.cpp:139-243)
    slots = ""
    if rng.random() < 0.5:
        groups = [f"[{i}, {nin + i}]" for i in range(min(nin, nout))]
        slots = f" attributes {{stencil.time_slots = [{', '.join(groups)}]}}"
    L = [f"builtin.module{slots} {{", f"  func.func @step({', '.join(args)}) {{"]
    for i in range(nin):
        L.append(f"    %t{i} = stencil.load %in{i} : {ftype} -> !temp<?x{elem}>")
    names = [f"%a{i}" for i in range(nin)]
    opnds = ", ".join(f"%a{i} = %t{i} : !temp<?x{elem}>" for i in range(nin))
    res = ", ".join(f"%o{i}" for i in range(nout))
    rt = ", ".join([f"!temp<?x{elem}>"] * nout)
    L.append(f"    {res} = stencil.apply({opnds}) -> {'(' + rt + ')' if nout > 1 else rt} {{")
    L += _region(rng, names, nin, r, [h] * nin, rng.randint(4, 16), nout, "v", elem)
    L.append("    }")
    sb = _btxt([0] * r, n)
    for i in range(nout):
        L.append(f"    stencil.store %o{i} to %out{i} ({sb}) : !temp<?x{elem}> to {ftype}")
    L += ["    func.return", "  }", "}", ""]
    return "\n".join(L)


def multi_apply(seed: int):
    rng = random.Random(seed)
    r = rng.choice([2, 3])
    elem = rng.choice(["f32", "f32", "f64"])
    n = [rng.randint(5, 12) for _ in range(r)]
    h = 2
    fb = _btxt([-h] * r, [x + h for x in n])
    ftype = f"!field<{fb}x{elem}>"
    tt = f"!temp<?x{elem}>"
    args = [f"%u : {ftype}", f"%w : {ftype}", f"%o1 : {ftype}", f"%o2 : {ftype}"]
    L = [f"builtin.module {{", f"  func.func @step({', '.join(args)}) {{",
         f"    %tu = stencil.load %u : {ftype} -> {tt}",
         f"    %tw = stencil.load %w : {ftype} -> {tt}"]
    np_ = rng.randint(1, 2)
    pres = ", ".join(f"%p{i}" for i in range(np_))
    prt = ", ".join([tt] * np_)
    # producer: reads u with offsets <= 1 (its domain is the core widened by 1)
    L.append(f"    {pres} = stencil.apply(%a = %tu : {tt}, %b = %tw : {tt}) -> "
             f"{'(' + prt + ')' if np_ > 1 else prt} {{")
    L += _region(rng, ["%a", "%b"], 2, r, [1, 1], rng.randint(3, 10), np_, "x", elem)
    L.append("    }")
    # consumer: reads the producer's temps with offsets <= 1 and w with offsets <= 2
    cop = ", ".join([f"%c{i} = %p{i} : {tt}" for i in range(np_)] + [f"%d = %tw : {tt}"])
    L.append(f"    %q = stencil.apply({cop}) -> {tt} {{")
    L += _region(rng, [f"%c{i}" for i in range(np_)] + ["%d"], np_ + 1, r, [1] * np_ + [2],
                 rng.randint(3, 10), 1, "y", elem)
    L.append("    }")
    # independent third apply on u
    L.append(f"    %s = stencil.apply(%e = %tu : {tt}) -> {tt} {{")
    L += _region(rng, ["%e"], 1, r, [2], rng.randint(2, 8), 1, "z", elem)
    L.append("    }")
    sb = _btxt([0] * r, n)
    L.append(f"    stencil.store %q to %o1 ({sb}) : {tt} to {ftype}")
    L.append(f"    stencil.store %s to %o2 ({sb}) : {tt} to {ftype}")
    L += ["    func.return", "  }", "}", ""]
    return "\n".join(L)
