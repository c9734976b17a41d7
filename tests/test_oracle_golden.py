"""The C restatement oracle (oracle/hg_oracle.c) pinned against the reference's own outputs
(tests/golden/reference_golden.json, produced by the real reference core).  CPU only."""
import struct

import numpy as np
import pytest

from helpers import case_id, decomp_from_json, fp_hex, program_from_json


def test_init_values(golden, port):
    # exec::initValue (buffer.cpp:142-156), f64 bits and the f32 cast
    for iv in golden["init_values"]:
        v = port.init_value(iv["field"], iv["coord"])
        assert struct.pack("<d", v).hex() == iv["f64"], iv
        assert struct.pack("<f", v).hex() == iv["f32"], iv


def _serial_cases(golden, big=False):
    out = []
    for c in golden["serial"]:
        heavy = c["spec"][2] >= 1024 and c["T"] > 1
        if heavy == big:
            out.append(c)
    return out


def _run_case(port, c):
    prog = program_from_json(c["program"])
    arrays = port.initial_fields(prog)
    assert [fp_hex(a) for a in arrays] == c["init_fp"]
    perm = port.run(prog, arrays, c["T"])
    assert [fp_hex(arrays[p]) for p in perm] == c["final_fp"]


@pytest.mark.parametrize("idx", range(27))
def test_serial_runs_match_reference(golden, port, idx):
    cases = _serial_cases(golden)
    if idx >= len(cases):
        pytest.skip("no such case")
    _run_case(port, cases[idx])


def test_config1_full_run_matches_reference(golden, port):
    # heat 2D SDO2 1024^2 f32, T=100 -- BASELINE config 1, bitwise (survey fingerprints)
    (c,) = _serial_cases(golden, big=True)
    assert c["final_fp"] == ["b11e8dddf9e8c23c", "34a5556efc0dfea0"]
    _run_case(port, c)


def test_authored_programs(golden, port):
    for c in golden["authored"]:
        prog = program_from_json(c["program"])
        arrays = port.initial_fields(prog)
        assert [fp_hex(a) for a in arrays] == c["init_fp"], c["name"]
        perm = port.run(prog, arrays, c["T"])
        assert [fp_hex(arrays[p]) for p in perm] == c["final_fp"], c["name"]


def test_simulate_matches_reference(golden, port):
    import paper_2404_02218_b200 as hg
    for c in golden["decomposed"]:
        local = program_from_json(c["local_program"])
        dc = decomp_from_json(c["decomp"])
        # global init = initialFields of the undecomposed module
        k, r, e, o, f32 = c["spec"]
        glob = hg.Program.build(hg.KernelSpec(k, r, e, o, "f32" if f32 else "f64"))
        arrays = port.initial_fields(glob)
        lbs = [glob.field_bounds(i)[0] for i in range(glob.nfields)]
        outs = port.simulate(local, dc, arrays, lbs, c["T"])
        assert [fp_hex(a) for a in outs] == c["sim_fp"], case_id(c)
        assert c["sim_fp"] == c["serial_fp"] == c["mpi_sim_fp"]


def test_exchange_declarations(golden, port):
    for x in golden["dmp"]["exchanges"]:
        got = port.exchanges(x["core"], x["below"], x["above"], x["grid"], x["coord"])
        want = [{"at": d[0], "size": d[1], "offset": d[2], "to": d[3]} for d in x["decls"]]
        assert got == want, x


def test_listing2_exchange_layout(port):
    # dmp_tests.cpp:122-147 / fixtures/listing2.xir: 100x100 core, width-4 halos
    d = port.exchanges([100, 100], [4, 4], [4, 4])
    assert [e["to"] for e in d] == [[-1, 0], [1, 0], [0, -1], [0, 1]]
    assert d[0]["at"] == [0, 4] and d[0]["size"] == [4, 100] and d[0]["offset"] == [4, 0]
    assert d[1]["at"] == [104, 4] and d[1]["offset"] == [-4, 0]
    assert d[3]["at"] == [4, 104] and d[3]["size"] == [100, 4] and d[3]["offset"] == [0, -4]


def test_neighbors_and_slicing(golden, port):
    import ctypes as C
    L = port.L
    for n in golden["dmp"]["neighbors"]:
        k = len(n["grid"])
        got = L.or_neighbor_rank(k, n["rank"], (C.c_int64 * k)(*n["dir"]),
                                 (C.c_int64 * k)(*n["grid"]))
        assert got == n["nbr"], n
    for ext, parts, p, lb, ub in golden["dmp"]["slicing"]:
        a, b = C.c_int64(), C.c_int64()
        L.or_local_interval(ext, parts, p, C.byref(a), C.byref(b))
        assert (a.value, b.value) == (lb, ub)


def test_binding_after(golden, port):
    import ctypes as C
    for b in golden["binding_after"]:
        gl = (C.c_int32 * len(b["groups"]))(*[len(g) for g in b["groups"]])
        flat = [i for g in b["groups"] for i in g]
        gg = (C.c_int32 * len(flat))(*flat)
        out = (C.c_int32 * 16)()
        port.L.or_binding_after(len(b["groups"]), gl, gg, b["nargs"], b["steps"], out)
        assert list(out[:b["nargs"]]) == b["perm"]


def test_pack_unpack_roundtrip(port):
    # packRegion/unpackRegion are inverse row-major walks over the box (simulator.cpp:523-584)
    rng = np.random.default_rng(5)
    a = rng.standard_normal((7, 9, 11)).astype(np.float32)
    lb = [-2, -2, -2]
    at, size = [1, 2, 3], [4, 5, 6]
    packed = port.pack(a, lb, at, size)
    assert np.array_equal(packed, a[1:5, 2:7, 3:9].reshape(-1))
    b = np.zeros_like(a)
    port.unpack(b, lb, at, size, packed)
    assert np.array_equal(b[1:5, 2:7, 3:9], a[1:5, 2:7, 3:9])
    assert np.count_nonzero(b) == np.count_nonzero(a[1:5, 2:7, 3:9])


def test_decomposed_multi_apply(golden, port):
    # independent applies in one step, decomposed: a swap before every load (the reference's
    # decompose, dmp_transforms.cpp:276-300), simulate == serial == lowered-mpi simulate
    import paper_2404_02218_b200 as hg
    assert len(golden["decomposed_authored"]) >= 2
    for c in golden["decomposed_authored"]:
        glob = program_from_json(c["program"])
        local = program_from_json(c["local_program"])
        dc = decomp_from_json(c["decomp"])
        arrays = port.initial_fields(glob)
        assert [fp_hex(a) for a in arrays] == c["init_fp"], c["name"]
        lbs = [glob.field_bounds(i)[0] for i in range(glob.nfields)]
        outs = port.simulate(local, dc, arrays, lbs, c["T"])
        assert [fp_hex(a) for a in outs] == c["sim_fp"], c["name"]
        assert c["sim_fp"] == c["serial_fp"] == c["mpi_sim_fp"]
        assert isinstance(glob, hg.Program)


def test_apply_fusion_matches_reference(golden, port):
    # hg_fuse_applies: every authored multi-apply step fused into one apply reproduces the
    # reference's materialised run bit for bit (on the oracle)
    n = 0
    for c in golden["authored"]:
        if "applies" not in c["program"]:
            continue
        fused = program_from_json(c["program"]).fuse_applies()
        arrays = port.initial_fields(fused)
        perm = port.run(fused, arrays, c["T"])
        assert [fp_hex(arrays[p]) for p in perm] == c["final_fp"], c["name"]
        n += 1
    assert n >= 5
