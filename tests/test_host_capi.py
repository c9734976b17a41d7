"""Host side of the C-ABI (no GPU): the library loads and exports every symbol of
include/hg/hg.h; the program builder, decompose pass, dmp arithmetic, initializer and binding
rotation reproduce the reference's own outputs (tests/golden/) exactly; errors are loud."""
import ctypes as C
import struct

import numpy as np
import pytest

import paper_2404_02218_b200 as hg
from paper_2404_02218_b200 import _capi as capi
from helpers import decomp_to_json, program_from_json, prog_to_json


def test_library_exports_every_declared_symbol():
    L = capi.lib()
    names = capi.exported_symbols()
    assert len(names) >= 35
    for n in names:
        assert hasattr(L, n), n


def test_builder_matches_reference_modules(golden):
    # exec::buildKernel (kernels.cpp:139-243) re-read from the reference module, op by op,
    # including the f32 constant bits of the retyped module
    for c in golden["serial"]:
        k, r, e, o, f32 = c["spec"]
        p = hg.Program.build(hg.KernelSpec(k, r, e, o, "f32" if f32 else "f64"))
        assert prog_to_json(p) == c["program"], c["spec"]


def test_f32_constant_bits_from_survey():
    p = hg.Program.build(hg.KernelSpec("wave", 3, 16, 8, "f32"))
    bits = [o.bits for o in p.op_list() if o.code == capi.HG_OP_CONST]
    assert {0xc0fc0000, 0x3fb60b61, 0xbde38e39, 0x3ab60b61, 0x40000000, 0x3c23d70a} == set(bits)
    p = hg.Program.build(hg.KernelSpec("heat", 3, 16, 4, "f32"))
    bits = {o.bits for o in p.op_list() if o.code == capi.HG_OP_CONST}
    assert bits == {0xc0f00000, 0x3faaaaab, 0xbdaaaaab, 0x3c23d70a}


def test_decompose_matches_reference(golden):
    # the decompose pass (dmp_transforms.cpp:101-312): local field bounds, stores, swaps
    for c in golden["decomposed"]:
        k, r, e, o, f32 = c["spec"]
        p = hg.Program.build(hg.KernelSpec(k, r, e, o, "f32" if f32 else "f64"))
        local, dc = p.decompose(c["grid"])
        assert prog_to_json(local) == c["local_program"], c["spec"]
        assert decomp_to_json(dc) == c["decomp"], c["spec"]


def test_decompose_rejects_what_the_reference_rejects():
    p = hg.Program.build(hg.KernelSpec("heat", 2, 10, 2, "f32"))
    with pytest.raises(capi.HgError, match="not divisible"):
        p.decompose([3, 1])
    with pytest.raises(capi.HgError, match="grid rank"):
        p.decompose([2])
    p = hg.Program.build(hg.KernelSpec("heat", 2, 4, 8, "f32"))
    with pytest.raises(capi.HgError, match="halo width exceeds"):
        p.decompose([2, 2])


def test_exchanges_neighbors_slicing_binding(golden):
    for x in golden["dmp"]["exchanges"]:
        got = hg.exchanges(x["core"], x["below"], x["above"], x["grid"], x["coord"])
        want = [{"at": d[0], "size": d[1], "offset": d[2], "to": d[3]} for d in x["decls"]]
        assert got == want
    for n in golden["dmp"]["neighbors"]:
        assert hg.neighbor_rank(n["rank"], n["dir"], n["grid"]) == n["nbr"]
    for c in golden["dmp"]["coords"]:
        assert hg.coord_from_rank(c["rank"], c["grid"]) == c["coord"]
        assert hg.rank_from_coord(c["coord"], c["grid"]) == c["rank"]
    for ext, parts, p, lb, ub in golden["dmp"]["slicing"]:
        assert hg.local_interval(ext, parts, p) == (lb, ub)
    for b in golden["binding_after"]:
        assert hg.binding_after(b["groups"], b["nargs"], b["steps"]) == b["perm"]


def test_init_value_and_fingerprint(golden):
    for iv in golden["init_values"]:
        v = hg.init_value(iv["field"], iv["coord"])
        assert struct.pack("<d", v).hex() == iv["f64"]
    assert hg.fingerprint(np.zeros(0, np.uint8)) == 0xcbf29ce484222325
    assert hg.fingerprint(np.frombuffer(b"a", np.uint8)) == 0xaf63dc4c8601ec8c  # FNV-1a("a")


def test_kernel_family_matching(golden):
    fam = {}
    for c in golden["serial"]:
        k, r, e, o, f32 = c["spec"]
        p = hg.Program.build(hg.KernelSpec(k, r, e, o, "f32" if f32 else "f64"))
        fam[(k, r, o, f32)] = p.kernel_family()
    assert fam[("heat", 3, 4, 1)] == "star3d_r2_heat_f32"
    assert fam[("wave", 3, 8, 1)] == "star3d_r4_wave_f32"
    assert fam[("heat", 2, 2, 1)] == "star2d_r1_heat_f32"
    assert fam[("heat", 3, 8, 0)] == "star3d_r4_heat_f64"
    assert fam[("heat", 1, 2, 1)] == "generic1d_f32"
    for c in golden["authored"]:
        fam = program_from_json(c["program"]).kernel_family()
        assert fam.startswith("multi" if "applies" in c["program"] else "generic"), fam


def test_validation_errors():
    p = hg.Program.build(hg.KernelSpec("heat", 2, 8, 2, "f32"))
    p.prog.ops[5].a = 7  # use before def
    with pytest.raises(capi.HgError, match="use before def"):
        p.kernel_family()
    p = hg.Program.build(hg.KernelSpec("heat", 2, 8, 2, "f32"))
    p.prog.ops[3].off[0] = 5  # reaches past the halo
    with pytest.raises(capi.HgError, match="escapes"):
        p.kernel_family()
    with pytest.raises(capi.HgError, match="unknown kernel"):
        hg.Program.build(hg.KernelSpec("nope", 2, 8, 2))
    with pytest.raises(capi.HgError, match="order"):
        hg.Program.build(hg.KernelSpec("heat", 2, 8, 3))


def test_plan_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    p = hg.Program.build(hg.KernelSpec("heat", 2, 8, 2, "f32"))
    with pytest.raises(capi.HgError) as e:
        hg.Plan(p)
    assert e.value.status == capi.HG_ECUDA


def test_csv_and_throughput():
    assert hg.csv_header() == "label,core_points,steps,seconds,gpts_per_s"
    assert hg.gpts_per_sec(10**9, 2, 4.0) == 0.5
    assert hg.csv_row("x", 100, 2, 0.5).startswith("x,100,2,0.5,")


def test_fused_apply_family_generates_and_compiles(golden):
    # NVRTC compiles the generated straight-line kernel for sm_100a (no GPU needed)
    import ctypes as C
    done = 0
    for c in golden["authored"]:
        p = program_from_json(c["program"])
        buf = C.create_string_buffer(1 << 20)
        n = C.c_size_t()
        rc = capi.lib().hg_apply_compile(C.byref(p.prog), buf, 1 << 20, C.byref(n))
        if p.rank == 1 or "applies" in c["program"]:
            assert rc == capi.HG_EUNSUPPORTED
            continue
        assert rc == 0, capi.lib().hg_last_error()
        assert n.value > 1000 and b"hg_apply" in buf.value
        assert b"__fadd_rn" in buf.value or b"__dadd_rn" in buf.value
        # one persistent wave walks the units, the TMA ring running across them
        assert b"u < P.units; u += gridDim.x" in buf.value
        done += 1
    assert done >= 4


@pytest.mark.parametrize("pack", ["0", "1"])
def test_fused_apply_pw_codegen(monkeypatch, pack):
    # the PW set (config 4) through both codegens: scalar, and f32 adds as FADD2 lanes with
    # scalar products (HG_JIT_PACK=1); both compile for sm_100a
    import ctypes as C
    monkeypatch.setenv("HG_JIT_PACK", pack)
    p = hg.Program.pw_advection(32, 64, 64)
    buf = C.create_string_buffer(1 << 21)
    n = C.c_size_t()
    assert capi.lib().hg_apply_compile(C.byref(p.prog), buf, 1 << 21, C.byref(n)) == 0, \
        capi.lib().hg_last_error()
    src = buf.value
    assert n.value > 1000
    assert (b"upk2(add2(pk2(" in src) == (pack == "1")
    assert b"mul.rn.f32x2" not in src  # products are never packed (no FFMA2 contraction)


def test_pw_advection_program():
    p = hg.Program.pw_advection(128, 512, 512)
    assert p.prog.nresults == 3 and p.prog.noperands == 3 and p.prog.nfields == 6
    assert p.core_points() == 128 * 512 * 512
    with pytest.raises(capi.HgError, match="diagonal"):
        p.decompose([2, 1, 1])


def test_no_fma_in_stencil_kernels():
    # the bit-exactness contract (no FMA contraction, proj/CMakeLists.txt:8-10) checked on the
    # shipped SASS: the star and resident kernels carry no FFMA/DFMA/FFMA2 at all -- their f32
    # adds run as FADD2 lanes next to scalar FMULs, which ptxas must not fuse; only the generic
    # kernel's correctly rounded division (__fdiv_rn/__ddiv_rn expansion) may use fused steps
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    sass = subprocess.run(["cuobjdump", "-sass", capi.LIB_PATH], capture_output=True,
                          text=True).stdout
    fn, bad, seen, packed = None, [], 0, 0
    for line in sass.splitlines():
        if "Function :" in line:
            fn = line.split("Function :")[1].strip()
            seen += "starKernel" in fn or "residentKernel" in fn
        # (HFMA2 Rx, -RZ, RZ, imm is ptxas' constant-materialisation idiom, not arithmetic)
        elif fn and ("starKernel" in fn or "residentKernel" in fn):
            if any(op in line for op in ("FFMA", "DFMA")):
                bad.append((fn, line.strip()))
            packed += "FADD2" in line
    assert seen >= 30
    assert packed > 0  # the f32 instances do run packed adds
    assert not bad, bad[:3]


def test_native_xir_reader_matches_reference_parser(golden):
    # hg_parse_program reads the reference's printed modules into the same descriptors the
    # reference's own parser + IR walk produce (serial, authored, decomposed + swaps)
    n = 0
    for c in golden["serial"] + golden["authored"]:
        if not c.get("text"):
            continue
        prog, dc, _ = hg.Program.parse(c["text"])
        assert prog_to_json(prog) == c["program"], c.get("name", c.get("spec"))
        assert dc is None
        n += 1
    for c in golden["decomposed"]:
        prog, dc, reftext = hg.Program.parse(c["text"])
        assert prog_to_json(prog) == c["local_program"]
        assert decomp_to_json(dc) == c["decomp"]
        glob, _, _ = hg.Program.parse(reftext)        # the dmp.reference snapshot
        assert glob.core_points() == prog.core_points() * int(np.prod(c["grid"]))
        n += 1
    assert n >= 30


def test_native_xir_reader_errors():
    with pytest.raises(capi.HgError, match="<xir>:1:1"):
        hg.Program.parse("module {}")
    bad = ("builtin.module {\n  func.func @f(%a : !field<[0,4]xf32>, %b : !field<[0,4]xf32>) {\n"
           "    %t = stencil.load %a : !field<[0,4]xf32> -> !temp<?xf32>\n"
           "    %o = stencil.apply(%x = %t : !temp<?xf32>) -> !temp<?xf32> {\n"
           "      %v = arith.addf %x, %x : f32\n      stencil.return %v : f32\n    }\n")
    with pytest.raises(capi.HgError, match="use before def"):
        hg.Program.parse(bad)


def test_decompose_multi_apply_matches_reference(golden):
    # our decompose on the multi-apply descriptor == the reference's pass (local program with
    # rewritten apply domains, one swap per load in load order)
    for c in golden["decomposed_authored"]:
        glob = program_from_json(c["program"])
        local, dc = glob.decompose(c["grid"])
        assert prog_to_json(local) == c["local_program"], c["name"]
        assert decomp_to_json(dc) == c["decomp"], c["name"]
        prog, pdc, ref = hg.Program.parse(c["text"])          # the printed dmp-level module
        assert prog_to_json(prog) == c["local_program"]
        assert decomp_to_json(pdc) == c["decomp"]
        g2, _, _ = hg.Program.parse(ref)
        assert prog_to_json(g2) == c["program"]


def test_decompose_rejects_chained_applies(golden):
    for c in golden["authored"]:
        j = c["program"]
        if "applies" not in j or not any(x < 0 for a in j["applies"] for x in a["operands"]):
            continue
        p = program_from_json(j)
        grid = [1] * p.rank
        with pytest.raises(capi.HgError, match="apply consuming another apply"):
            p.decompose(grid)
