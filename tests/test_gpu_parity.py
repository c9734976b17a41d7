"""GPU parity: the sm_100a path (through the C-ABI) against the reference's own outputs
(tests/golden/, bitwise FNV-1a fingerprints) and against the C restatement oracle on the same
seeded inputs.  Bar: bit-exact fields, halos included (the reference evaluates a fixed IEEE op
DAG with no FMA, proj/CMakeLists.txt:8-10; the stated fallback tolerance, max relative error
<= 1e-5, is never needed and never used here)."""
import ctypes as C

import numpy as np
import pytest

import paper_2404_02218_b200 as hg
from helpers import case_id, decomp_from_json, fp_hex, program_from_json

pytestmark = pytest.mark.gpu


def _plan_run(prog, T):
    plan = hg.Plan(prog)
    plan.init_fields()
    init = [plan.download(i) for i in range(prog.nfields)]
    plan.run(T)
    perm, steps = plan.binding()
    assert steps == T
    fin = [plan.download(p) for p in perm]
    name = plan.kernel_name
    plan.close()
    return init, fin, perm, name


def _serial(golden, big=False):
    return [c for c in golden["serial"] if (c["spec"][2] >= 1024 and c["T"] > 1) == big]


def test_serial_cases_bitwise(golden):
    seen = set()
    for c in _serial(golden):
        prog = program_from_json(c["program"])
        init, fin, perm, name = _plan_run(prog, c["T"])
        seen.add(name.replace("+resident", ""))
        assert [fp_hex(a) for a in init] == c["init_fp"], case_id(c)
        assert [fp_hex(a) for a in fin] == c["final_fp"], (case_id(c), name)
    # both families and every tap radius were exercised
    assert {"star2d_r1_heat_f32", "star3d_r2_heat_f32", "star3d_r4_wave_f32",
            "star3d_r4_heat_f64", "generic1d_f32"} <= seen


@pytest.mark.parametrize("path", ["resident", "star"])
def test_config1_full_run_bitwise(golden, monkeypatch, path):
    # BASELINE config 1 end to end against the reference's own fingerprints: the whole run in
    # one shared-memory-resident launch (default) and step by step through the star kernel
    if path == "star":
        monkeypatch.setenv("HG_NO_RESIDENT", "1")
    (c,) = _serial(golden, big=True)
    prog = program_from_json(c["program"])
    _, fin, _, name = _plan_run(prog, c["T"])
    assert name == "star2d_r1_heat_f32" + ("+resident" if path == "resident" else "")
    assert [fp_hex(a) for a in fin] == ["b11e8dddf9e8c23c", "34a5556efc0dfea0"]


@pytest.mark.parametrize("family", ["apply", "generic", "unfused"])
def test_authored_programs_bitwise(golden, monkeypatch, family):
    # multi-operand / multi-result / divide / diagonal programs incl. the authored
    # PW-advection set: the fused-apply family (NVRTC-generated) and the generic kernel;
    # multi-apply steps fused (default) or apply by apply ("unfused")
    if family == "generic":
        monkeypatch.setenv("HG_NO_APPLY_JIT", "1")
    if family == "unfused":
        monkeypatch.setenv("HG_NO_FUSE_APPLIES", "1")
    for c in golden["authored"]:
        prog = program_from_json(c["program"])
        init, fin, _, name = _plan_run(prog, c["T"])
        want = ("multi" if "applies" in c["program"] else
                "apply" if family == "unfused" and prog.rank >= 2 else
                family if prog.rank >= 2 else "generic")
        assert name.startswith(want), (c["name"], name)
        assert [fp_hex(a) for a in init] == c["init_fp"], c["name"]
        assert [fp_hex(a) for a in fin] == c["final_fp"], c["name"]


def test_pw_advection_config4_against_oracle(port):
    # BASELINE config 4 shape: 128 x 512 x 512 (x fastest), bitwise incl. the halo rims
    prog = hg.Program.pw_advection(128, 512, 512)
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, 1)
    init, fin, perm, name = _plan_run(prog, 1)
    assert name == "apply3d_f32" and perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


@pytest.mark.parametrize("spec,T", [(("wave", 3, 45, 4), 4), (("heat", 3, 70, 8), 3),
                                    (("heat", 2, 300, 2), 5)])
def test_apply_family_on_star_programs_matches(port, monkeypatch, spec, T):
    # the generated family also runs the generator's kernels bit-exactly
    monkeypatch.setenv("HG_NO_STAR", "1")
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    _, fin, perm, name = _plan_run(prog, T)
    assert name.startswith("apply") and perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_run_serial_stencil_host_api(port):
    # exec::runSerialStencil semantics: caller buffers updated in place, result = final binding
    prog = hg.build_kernel(hg.KernelSpec("wave", 3, 37, 8, "f32"))
    arrays = port.initial_fields(prog)
    bufs = [hg.Buffer(a.copy(), prog.field_bounds(i)[0]) for i, a in enumerate(arrays)]
    out = hg.run_serial_stencil(prog, bufs, 5)
    perm = port.run(prog, arrays, 5)
    assert [id(b) for b in out] == [id(bufs[p]) for p in perm]
    for b, p in zip(out, perm):
        assert np.array_equal(b.data.view(np.uint32), arrays[p].view(np.uint32))


def test_split_runs_equal_one_run():
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 70, 4, "f32"))
    a = hg.Plan(prog)
    b = hg.Plan(prog)
    a.init_fields()
    b.init_fields()
    a.run(7)
    for _ in range(7):
        b.run(1)
    assert a.binding() == b.binding()
    for i in range(prog.nfields):
        assert fp_hex(a.download(i)) == fp_hex(b.download(i))


@pytest.mark.parametrize("spec,T", [
    (("heat", 3, 256, 4), 3), (("wave", 3, 160, 8), 3), (("heat", 3, 131, 8), 2),
    (("wave", 2, 1000, 2), 5), (("heat", 2, 777, 8), 4), (("wave", 3, 99, 2), 4),
])
def test_against_oracle_medium(port, spec, T):
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    init, fin, perm, _ = _plan_run(prog, T)
    assert perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


@pytest.mark.slow
def test_config2_shape_against_oracle(port):
    # BASELINE config 2 shape (heat 3D SDO4 512^3), T=2, bitwise incl. halos
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 512, 4, "f32"))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, 2)
    _, fin, perm, name = _plan_run(prog, 2)
    assert name == "star3d_r2_heat_f32" and perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


def test_pack_unpack_match_oracle(port):
    import torch
    rng = np.random.default_rng(11)
    for spec in (("heat", 3, 21, 4), ("wave", 2, 40, 8), ("heat", 1, 30, 2)):
        prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
        plan = hg.Plan(prog)
        plan.init_fields()
        host = plan.download(0)
        lb = prog.field_bounds(0)[0]
        for _ in range(6):
            at = [int(rng.integers(0, s - 1)) for s in host.shape]
            size = [int(rng.integers(1, s - a + 1)) for a, s in zip(at, host.shape)]
            want = port.pack(host, lb, at, size)
            dev = torch.empty(want.size, dtype=torch.float32, device="cuda")
            plan.pack(0, at, size, dev.data_ptr())
            torch.cuda.synchronize()
            assert np.array_equal(dev.cpu().numpy().view(np.uint32), want.view(np.uint32))
            # unpack a pattern and compare with the oracle's unpack
            pat = (np.arange(want.size, dtype=np.float32) + 0.5)
            plan.unpack(1, at, size, torch.from_numpy(pat).cuda().data_ptr())
            torch.cuda.synchronize()
            exp = plan.download(1)  # device state after unpack
            ref1 = exp.copy()
            port.unpack(ref1, lb, at, size, pat)
            assert np.array_equal(exp, ref1)
        plan.close()


def test_simulate_matches_reference(golden):
    # exec::simulate over one process: decompose, scatter, device swaps, gather -- bitwise
    for c in golden["decomposed"]:
        k, r, e, o, f32 = c["spec"]
        prog = hg.build_kernel(hg.KernelSpec(k, r, e, o, "f32" if f32 else "f64"))
        init = hg.initial_fields(prog)
        out = hg.simulate(prog, c["grid"], init, c["T"], devices=[0] * int(np.prod(c["grid"])))
        assert [fp_hex(b.data) for b in out] == c["sim_fp"], case_id(c)


def test_simulate_multi_apply_matches_reference(golden, port):
    # decomposed multi-apply steps (independent applies, a swap before every load): gathered
    # result == the reference's simulate, and every rank's halos == the oracle's
    for c in golden["decomposed_authored"]:
        glob = program_from_json(c["program"])
        init = hg.initial_fields(glob)
        n = int(np.prod(c["grid"]))
        out = hg.simulate(glob, c["grid"], init, c["T"], devices=[0] * n)
        assert [fp_hex(b.data) for b in out] == c["sim_fp"], c["name"]
        local, dc, states = _sim_rank_states(glob, c["grid"], c["T"])
        arrays = port.initial_fields(glob)
        lbs = [glob.field_bounds(i)[0] for i in range(glob.nfields)]
        for rk in range(n):
            want = port.simulate_rank_state(local, dc, arrays, lbs, c["T"], rk)
            for g, o in zip(states[rk], want):
                assert np.array_equal(g.view(np.uint8), o.view(np.uint8)), (c["name"], rk)


def _sim_rank_states(prog, grid, T):
    """Run simulate's loop and return every rank's local buffers (halos included) in final
    binding order."""
    local, dc = prog.decompose(grid)
    n = int(np.prod(grid))
    plans, dmps = [], []
    for rk in range(n):
        pl = hg.Plan(local)
        coord = hg.coord_from_rank(rk, grid)
        pl.init_fields(origin=[coord[d] * dc.core[d] for d in range(prog.rank)])
        plans.append(pl)
        dmps.append(hg.Dmp(pl, dc, rk))
    arr = (C.c_void_p * n)(*[d.h for d in dmps])
    hg.check(hg.lib().hg_sim_connect(arr, n))
    hg.check(hg.lib().hg_sim_run(arr, n, T, None))
    states = []
    for rk in range(n):
        perm, _ = plans[rk].binding()
        states.append([plans[rk].download(p) for p in perm])
    for d in dmps:
        d.close()
    for p in plans:
        p.close()
    return local, dc, states


@pytest.mark.parametrize("spec,grid,T", [
    (("heat", 3, 16, 4), [2, 2, 2], 3), (("wave", 3, 24, 8), [3, 1, 2], 4),
    (("heat", 2, 30, 2), [3, 2], 5), (("wave", 2, 40, 4), [2, 4], 3),
    (("heat", 3, 32, 2), [4, 1, 1], 2),
    (("heat", 3, 32, 4), [2, 4, 1], 3),  # the N=8 strong grid (strong_grid(8))
])
def test_rank_halos_bitwise_after_swaps(port, spec, grid, T):
    # per-rank local state (cores AND halos) == the oracle's restatement of RankHooks::swap
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    local, dc, states = _sim_rank_states(prog, grid, T)
    glob = port.initial_fields(prog)
    lbs = [prog.field_bounds(i)[0] for i in range(prog.nfields)]
    for rk, st in enumerate(states):
        want = port.simulate_rank_state(local, dc, glob, lbs, T, rk)
        for g, w in zip(st, want):
            assert np.array_equal(g.view(np.uint32), w.view(np.uint32)), (spec, grid, rk)


# ---- two-step passes (temporal blocking, tb.cu) ----------------------------------------------
def _tb_case(port, prog, calls, upload_rng=None):
    """Run `calls` (a list of step counts) through one plan and compare every buffer, halos
    included, with the oracle; optionally upload random fields (rings included) first."""
    plan = hg.Plan(prog)
    plan.init_fields()
    arrays = [plan.download(i) for i in range(prog.nfields)]
    if upload_rng is not None:
        plan.run(2)                 # make the plan own shadows, then replace the data
        plan.reset_binding()
        arrays = [upload_rng.random(a.shape, dtype=np.float32) for a in arrays]
        for i, a in enumerate(arrays):
            plan.upload(i, a)
    l0 = plan.launch_count()
    for c in calls:
        plan.run(c)
    launches = plan.launch_count() - l0
    perm, _ = plan.binding()
    got = [plan.download(p) for p in perm]
    plan.close()
    T = sum(calls)
    perm_o = port.run(prog, arrays, T)
    assert perm == perm_o
    for g, o in zip(got, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))
    return launches


@pytest.mark.parametrize("order,ext,calls", [
    (4, [130, 200, 250], [4]), (4, [130, 200, 250], [5]), (4, [96, 160, 360], [3, 2, 1]),
    (2, [100, 210, 243], [6]), (2, [171, 171, 171], [1, 4]), (4, [256, 64, 300], [2]),
])
def test_two_step_passes_bitwise(port, monkeypatch, order, ext, calls):
    # heat 3D star, > 4M points: pairs of steps per pass, ragged tiles in x (not a multiple of
    # the 120-point tile or of 4) and y, odd counts ending in one ordinary step, split calls
    monkeypatch.setenv("HG_TB", "1")
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, order, "f32")).with_extents(ext)
    launches = _tb_case(port, prog, calls)
    assert launches == sum(c // 2 + c % 2 for c in calls)


def test_two_step_passes_after_upload(port, monkeypatch):
    # uploads replace the rings too: the shadow of a buffer must follow
    monkeypatch.setenv("HG_TB", "1")
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents([140, 180, 200])
    _tb_case(port, prog, [4, 3], upload_rng=np.random.default_rng(7))


def test_two_step_matches_single_step(monkeypatch):
    # the same run with passes disabled: identical buffers (and the same binding)
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 176, 4, "f32"))
    outs = []
    for on in (True, False):
        monkeypatch.setenv("HG_TB", "1" if on else "0")
        plan = hg.Plan(prog)
        plan.init_fields()
        plan.run(6)
        perm, _ = plan.binding()
        outs.append((perm, [plan.download(p) for p in perm], plan.launch_count()))
        plan.close()
    assert outs[0][0] == outs[1][0]
    for a, b in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


# ---- two output rows per thread (GEO 3, 128 x 16 tile) ------------------------------------------
@pytest.mark.parametrize("order,ext,T", [
    (4, [24, 16, 128], 3),    # one tile, one chunk
    (4, [40, 37, 140], 3),    # ragged y (odd: a thread's second row past the domain), ragged x
    (2, [30, 33, 200], 4),    # SDO2 (radius 1)
    (4, [300, 50, 260], 2),   # several z-chunks (L2 hints), ragged y and x
    (4, [36, 800, 1000], 2),  # the benched plane shape class
])
def test_two_row_tile_bitwise(port, monkeypatch, order, ext, T):
    monkeypatch.setenv("HG_STAR_GEO", "3")
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, order, "f32")).with_extents(ext)
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    _, fin, perm, name = _plan_run(prog, T)
    assert name.startswith("star3d_r"), name
    assert perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


# ---- wide-tile geometry of the star kernel (large x-y planes) ---------------------------------
@pytest.mark.parametrize("order,ext,T", [(4, [36, 800, 1000], 3), (2, [20, 771, 903], 4)])
def test_wide_tile_geometry_bitwise(port, order, ext, T):
    # planes >= 768 x 768 take the 128 x 12 tile (starGeoFor); ragged in x and y
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, order, "f32")).with_extents(ext)
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    _, fin, perm, _ = _plan_run(prog, T)
    assert perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


@pytest.mark.parametrize("geo", ["1", "3"])
@pytest.mark.parametrize("spec,grid,T", [(("heat", 3, 24, 4), [2, 2, 1], 4),
                                         (("heat", 3, 32, 2), [1, 2, 2], 3)])
def test_wide_tile_rank_halos(port, monkeypatch, spec, grid, T, geo):
    # the wide tiles forced on small ranks: per-rank halos after device swaps stay bitwise
    monkeypatch.setenv("HG_STAR_GEO", geo)
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    local, dc, states = _sim_rank_states(prog, grid, T)
    glob = port.initial_fields(prog)
    lbs = [prog.field_bounds(i)[0] for i in range(prog.nfields)]
    for rk in range(int(np.prod(grid))):
        want = port.simulate_rank_state(local, dc, glob, lbs, T, rk)
        for g, o in zip(states[rk], want):
            assert np.array_equal(g.view(np.uint32), o.view(np.uint32)), rk


@pytest.mark.parametrize("family,prefix", [
    ("fused", "multi2x_fused_apply3d"), ("unfused", "multi2x_apply3d"),
    ("generic", "multi2x_generic3d"), ("fused_generic", "multi2x_fused_generic3d")])
def test_multi_apply_flux3d_medium(port, monkeypatch, family, prefix):
    # the authored two-stage flux step (apply consuming apply) at a medium ragged size: fused
    # into one generated kernel (temps inlined), apply by apply through HBM temps (consumer
    # stored in place), and both on the generic kernel
    from paper_2404_02218_b200.programs.flux3d import xir
    if family in ("unfused", "generic"):
        monkeypatch.setenv("HG_NO_FUSE_APPLIES", "1")
    if family in ("generic", "fused_generic"):
        monkeypatch.setenv("HG_NO_APPLY_JIT", "1")
    prog, _, _ = hg.Program.parse(xir(70, 130, 203))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, 3)
    _, fin, perm, name = _plan_run(prog, 3)
    assert name.startswith(prefix), name
    assert perm == perm_o
    for g, o in zip(fin, [arrays[p] for p in perm_o]):
        assert np.array_equal(g.view(np.uint32), o.view(np.uint32))


_SHALLOW_RING = r"""
import os, sys
import numpy as np
sys.path.insert(0, os.environ["REPO"]); sys.path.insert(0, os.path.join(os.environ["REPO"], "oracle"))
import paper_2404_02218_b200 as hg
from oracle import Port
from paper_2404_02218_b200.programs.flux3d import xir
from paper_2404_02218_b200.programs.pw_advection import xir as pw_xir
port = Port()
cases = [(hg.Program.parse(xir(12, 10, 21, "f64"))[0], 3),
         (hg.Program.parse(xir(7, 9, 8, "f64"))[0], 3),
         (hg.Program.parse(pw_xir(9, 10, 11, "f64"))[0], 2)]
bad = 0
for prog, T in cases:
    arrays = port.initial_fields(prog)
    want = [arrays[p] for p in port.run(prog, arrays, T)]
    for rep in range(8):
        plan = hg.Plan(prog); plan.init_fields(); plan.run(T)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
        plan.close()
        bad += sum(int(not np.array_equal(g.view(np.uint64), w.view(np.uint64)))
                   for g, w in zip(got, want))
print("bad", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("fuse", ["per-apply", "fused"])
def test_shallow_tma_ring_reuse_bitwise(fuse):
    # Stage-reuse hazard of the TMA ring: with a ring only one plane deeper than the stencil
    # window (HG_JIT_DEPTH=1) every stage is refilled while neighbouring warps still stream.
    # An arrive that did not follow the consumption of the loaded values let the refill land
    # before an f64 window's second LDS.128 had read it (failed every run before the fix).
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, REPO=repo, HG_JIT_DEPTH="1")
    if fuse == "per-apply":
        env["HG_NO_FUSE_APPLIES"] = "1"
    r = subprocess.run([sys.executable, "-c", _SHALLOW_RING], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("pinned", [True, False])
@pytest.mark.parametrize("spec,T,dtype", [
    (("heat", 3, 67, 4), 3, "f32"), (("wave", 3, 45, 8), 4, "f32"),
    (("heat", 2, 301, 2), 5, "f32"), (("heat", 3, 40, 2), 1, "f32"),
    (("heat", 3, 37, 4), 2, "f64"), (("heat", 2, 1023, 2), 4, "f32"),
    (("heat", 2, 203, 4), 3, "f64")])
def test_host_transfers_and_live_upload(port, pinned, spec, T, dtype):
    # uploads/downloads from pinned host memory (zero-copy kernel) and pageable memory (copy
    # engines); the live upload leaves the output slot's store box unmoved -- garbage there
    # must not matter, since step 1 overwrites it before anything reads it (2D heat cases
    # run through the resident whole-run kernel)
    import torch
    prog = hg.build_kernel(hg.KernelSpec(*spec, dtype))
    u = np.uint32 if dtype == "f32" else np.uint64
    arrays = port.initial_fields(prog)
    plan = hg.Plan(prog)
    try:
        # poison every buffer first, so a skipped region that mattered would show
        for i in range(prog.nfields):
            plan.upload(i, np.full_like(arrays[i], 1e30))
        hosts = []
        for i, a in enumerate(arrays):
            h = torch.from_numpy(a.copy()).pin_memory().numpy() if pinned else a.copy()
            hosts.append(h)
            plan.upload(i, h, live=True)
        # a full upload of buffer 0 round-trips exactly
        back = plan.download(0)
        assert np.array_equal(back.view(u), arrays[0].view(u))
        plan.run(T)
        perm, _ = plan.binding()
        outs = []
        for p in perm:
            o = np.empty_like(arrays[p])
            if pinned:
                o = torch.from_numpy(o).pin_memory().numpy()
            outs.append(plan.download(p, o))
    finally:
        plan.close()
    perm_o = port.run(prog, arrays, T)
    assert perm == perm_o
    for g, p in zip(outs, perm_o):
        assert np.array_equal(g.view(u), arrays[p].view(u))


@pytest.mark.parametrize("spec,T", [
    (("heat", 2, 1024, 2), 1), (("heat", 2, 1024, 2), 7), (("heat", 2, 1024, 2), 13),
    (("heat", 2, 1000, 4), 9), (("heat", 2, 777, 8), 6), (("heat", 2, 37, 2), 11),
    (("heat", 2, 300, 8), 3), (("heat", 2, 5, 2), 4)])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_resident_2d_bitwise(port, spec, T, dtype):
    # the shared-memory-resident whole-run kernel: bands, temporal blocks of K steps with the
    # boundary-row exchange between them, ragged last blocks and row/column tails, both
    # buffers' halo rings -- bitwise against the oracle, and split calls equal one call
    prog = hg.build_kernel(hg.KernelSpec(*spec, dtype))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    plan = hg.Plan(prog)
    try:
        plan.init_fields()
        assert plan.kernel_name.endswith("+resident"), plan.kernel_name
        plan.run(T)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
        plan.init_fields()
        plan.reset_binding()
        plan.run(T // 2)
        plan.run(T - T // 2)
        perm2, _ = plan.binding()
        got2 = [plan.download(p) for p in perm2]
    finally:
        plan.close()
    assert perm == perm_o == perm2
    u = np.uint32 if dtype == "f32" else np.uint64
    for g, g2, p in zip(got, got2, perm_o):
        assert np.array_equal(g.view(u), arrays[p].view(u))
        assert np.array_equal(g2.view(u), arrays[p].view(u))


def test_pageable_staged_transfers(port):
    # fields >= 32 MB in pageable host memory go through the pinned staging ring (chunks of
    # rows, multi-threaded host copies overlapped with the transfers): round trip and a run
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 300, 4, "f32"))  # 304^3 f32 = 112 MB
    arrays = port.initial_fields(prog)
    plan = hg.Plan(prog)
    try:
        for i, a in enumerate(arrays):
            plan.upload(i, a.copy(), live=(i == 1))
        back = plan.download(0)
        assert np.array_equal(back.view(np.uint32), arrays[0].view(np.uint32))
        plan.run(2)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
    finally:
        plan.close()
    perm_o = port.run(prog, arrays, 2)
    assert perm == perm_o
    for g, p in zip(got, perm_o):
        assert np.array_equal(g.view(np.uint32), arrays[p].view(np.uint32))


@pytest.mark.parametrize("spec", [("heat", 2, 64, 2), ("heat", 3, 40, 4), ("wave", 3, 24, 8)])
def test_zero_steps_leave_fields_and_binding(port, spec):
    # runSerialStencil with timesteps = 0 (serial.cpp:57-88): no step, identity binding; a
    # later run continues from the untouched fields (resident, star and wave paths)
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    arrays = port.initial_fields(prog)
    plan = hg.Plan(prog)
    try:
        plan.init_fields()
        plan.run(0)
        perm, steps = plan.binding()
        assert steps == 0 and perm == list(range(prog.nfields))
        for i, a in enumerate(arrays):
            assert np.array_equal(plan.download(i).view(np.uint32), a.view(np.uint32))
        plan.run(3)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
    finally:
        plan.close()
    perm_o = port.run(prog, arrays, 3)
    assert perm == perm_o
    for g, p in zip(got, perm_o):
        assert np.array_equal(g.view(np.uint32), arrays[p].view(np.uint32))


def test_live_upload_multi_apply(port):
    # hg_plan_upload_live on a multi-apply step: the skipped box is the stencil.store region
    # of the output field (mstore), over poisoned device buffers
    from paper_2404_02218_b200.programs.flux3d import xir
    prog = hg.Program.parse(xir(20, 18, 37))[0]
    arrays = port.initial_fields(prog)
    plan = hg.Plan(prog)
    try:
        for i in range(prog.nfields):
            plan.upload(i, np.full_like(arrays[i], np.float32(1e30)))
        import torch
        for i, a in enumerate(arrays):
            plan.upload(i, torch.from_numpy(a.copy()).pin_memory().numpy(), live=True)
        plan.run(3)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
    finally:
        plan.close()
    perm_o = port.run(prog, arrays, 3)
    assert perm == perm_o
    for g, p in zip(got, perm_o):
        assert np.array_equal(g.view(np.uint32), arrays[p].view(np.uint32))


@pytest.mark.parametrize("spec,T", [(("heat", 3, 70, 4), 3), (("wave", 3, 40, 8), 4),
                                    (("heat", 2, 300, 2), 5)])
def test_caller_bound_device_fields(port, spec, T):
    # hg_plan_bind: the fields live in the caller's device memory (torch tensors
    # here, laid out as hg_plan_layout says); init, steps and downloads go through them, and the
    # caller sees the results in its own tensors without a copy
    import torch
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    arrays = port.initial_fields(prog)
    perm_o = port.run(prog, arrays, T)
    plan = hg.Plan(prog)
    try:
        owned = []
        for b in range(prog.nfields):
            L = plan.layout(b)
            nbytes = L.pitch * L.rows * L.elem_bytes
            t = torch.empty(nbytes // 4 + 32, dtype=torch.float32, device="cuda")
            off = (-t.data_ptr()) % 128 // 4  # 128-byte aligned start inside the tensor
            owned.append((t, off, L))
            plan.bind(b, t.data_ptr() + 4 * off, nbytes)
        plan.init_fields()
        plan.run(T)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
        torch.cuda.synchronize()
        # the caller's own tensor holds the final field (its core rows at col0 of each row)
        t, off, L = owned[perm[0]]
        lo, hi = prog.field_bounds(perm[0])
        shape = [u - l for l, u in zip(lo, hi)]
        raw = t[off:off + L.pitch * L.rows].view(L.rows, L.pitch)[:, L.col0:L.col0 + shape[-1]]
        assert np.array_equal(raw.cpu().numpy().reshape(shape).view(np.uint32),
                              arrays[perm_o[0]].view(np.uint32))
    finally:
        plan.close()
    assert perm == perm_o
    for g, p in zip(got, perm_o):
        assert np.array_equal(g.view(np.uint32), arrays[p].view(np.uint32))
