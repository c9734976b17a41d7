"""Test helpers: golden-fixture programs -> hg descriptors."""
import ctypes as C

import numpy as np

import paper_2404_02218_b200 as hg
from paper_2404_02218_b200 import _capi as capi


def program_from_json(j) -> "hg.Program":
    return hg.Program.from_json(j)


def decomp_from_json(j) -> capi.HgDecomp:
    dc = capi.HgDecomp()
    n = len(j["grid"])
    dc.ndim = n
    for d in range(n):
        dc.grid[d] = j["grid"][d]
        dc.core[d] = j["core"][d]
    dc.nswaps = len(j["swaps"])
    for s, sw in enumerate(j["swaps"]):
        dc.swaps[s].field = sw["field"]
        dc.swaps[s].nexchanges = len(sw["ex"])
        for k, (at, size, off, to) in enumerate(sw["ex"]):
            e = dc.swaps[s].ex[k]
            for d in range(n):
                e.at[d], e.size[d], e.offset[d], e.to[d] = at[d], size[d], off[d], to[d]
    return dc


def prog_to_json(prog: "hg.Program"):
    p = prog.prog
    r = p.rank
    if p.napplies > 0:
        aps = p.applies
        return {
            "rank": r, "dtype": p.dtype, "nfields": p.nfields,
            "fields": [[list(p.fields[i].lb[:r]), list(p.fields[i].ub[:r])]
                       for i in range(p.nfields)],
            "ops": [[o.code, o.a, o.b, o.operand, list(o.off[:r]), "%016x" % o.bits]
                    for o in prog.op_list()],
            "applies": [{"operands": list(aps[a].operand[:aps[a].noperands]),
                         "op_begin": aps[a].op_begin, "nops": aps[a].nops,
                         "result_op": list(aps[a].result_op[:aps[a].nresults]),
                         "result_temp": list(aps[a].result_temp[:aps[a].nresults]),
                         "domain": [list(aps[a].domain.lb[:r]), list(aps[a].domain.ub[:r])]}
                        for a in range(p.napplies)],
            "loads": list(p.operand_field[:p.noperands]),
            "ntemps": p.ntemps,
            "mstores": [[p.mstore_temp[k], p.mstore_field[k], list(p.mstore[k].lb[:r]),
                         list(p.mstore[k].ub[:r])] for k in range(p.nstores)],
            "groups": prog.groups(),
        }
    return {
        "rank": r, "dtype": p.dtype, "nfields": p.nfields,
        "fields": [[list(p.fields[i].lb[:r]), list(p.fields[i].ub[:r])] for i in range(p.nfields)],
        "operand_field": list(p.operand_field[:p.noperands]),
        "ops": [[o.code, o.a, o.b, o.operand, list(o.off[:r]), "%016x" % o.bits]
                for o in prog.op_list()],
        "result_op": list(p.result_op[:p.nresults]),
        "store_field": list(p.store_field[:p.nresults]),
        "store": [[list(p.store[k].lb[:r]), list(p.store[k].ub[:r])] for k in range(p.nresults)],
        "groups": prog.groups(),
    }


def decomp_to_json(dc):
    n = dc.ndim
    return {"grid": list(dc.grid[:n]), "core": list(dc.core[:n]),
            "swaps": [{"field": s.field,
                       "ex": [[list(e.at[:n]), list(e.size[:n]), list(e.offset[:n]), list(e.to[:n])]
                              for e in s.ex[:s.nexchanges]]}
                      for s in dc.swaps[:dc.nswaps]]}


def fp_hex(arr: np.ndarray) -> str:
    return "%016x" % hg.fingerprint(arr)


def case_id(c):
    if "name" in c:
        return c["name"]
    k, r, e, o, f32 = c["spec"]
    s = f"{k}{r}d_n{e}_o{o}_{'f32' if f32 else 'f64'}"
    if "grid" in c:
        s += "_g" + "x".join(map(str, c["grid"]))
    return s + f"_T{c['T']}"
