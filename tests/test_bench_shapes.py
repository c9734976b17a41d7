"""GPU parity at the shapes the bench actually times ("What's weak" #1).

Every kernel instance behind a headline number is checked bit for bit against the C oracle
(oracle/hg_oracle.c, pinned to the reference by tests/golden/) on the same inputs:

* BASELINE config 5 at N=1 / config 2's kernel at full size: heat3d SDO4 1024^3, T=1 -- the
  wide 128x12 tile (GEO 1), 16 z-chunks, L2 eviction hints on the shared z-halo planes;
* BASELINE config 3: wave3d SDO8 1024^3, T=1 -- radius 4, 8 z-chunks, the depth-7 TMA ring;
* radius-4 multi-chunk cases at medium size (>= 3 chunks per column);
* a field of more than 2^31 elements (64-bit indexing end to end).

Reference semantics: exec::runSerialStencil (proj/core/src/exec/serial.cpp:57-88) over the
interpreter's stencil ops (interpreter.cpp:676-780).  Bar: bit-exact, halos included.

These need tens of GB of host memory for the oracle's fields; each case checks what the box
has first and skips (never swaps the box to death) when it is short.
"""
import numpy as np
import pytest

import paper_2404_02218_b200 as hg

pytestmark = pytest.mark.gpu


def _avail_bytes() -> int:
    try:
        import psutil
        return int(psutil.virtual_memory().available)
    except Exception:  # pragma: no cover
        import os
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")


def _field_bytes(prog) -> int:
    n = 0
    for i in range(prog.nfields):
        lo, hi = prog.field_bounds(i)
        m = 1
        for a, b in zip(lo, hi):
            m *= b - a
        n = max(n, m)
    return n * np.dtype(prog.dtype).itemsize


def _equal_chunked(a: np.ndarray, b: np.ndarray, what: str):
    """Bitwise equality of two large arrays without a full-size temporary; reports the first
    differing element."""
    assert a.shape == b.shape, what
    u = np.uint32 if a.itemsize == 4 else np.uint64
    fa, fb = a.reshape(-1).view(u), b.reshape(-1).view(u)
    step = 1 << 26
    for s in range(0, fa.size, step):
        x, y = fa[s:s + step], fb[s:s + step]
        if not np.array_equal(x, y):
            k = s + int(np.flatnonzero(x != y)[0])
            idx = np.unravel_index(k, a.shape)
            raise AssertionError(f"{what}: first difference at raw index {idx}: "
                                 f"{a.reshape(-1)[k]!r} vs {b.reshape(-1)[k]!r}")


def _big_case(port, prog, T, name_prefix):
    fb = _field_bytes(prog)
    # oracle fields + one apply temporary + one downloaded field, plus slack
    need = (prog.nfields + 2) * fb + (4 << 30)
    if _avail_bytes() < need:
        pytest.skip(f"needs ~{need / 2**30:.0f} GiB of free host memory")
    plan = hg.Plan(prog)
    try:
        plan.init_fields()
        plan.run(T)
        perm, steps = plan.binding()
        name = plan.kernel_name
        assert steps == T and name.startswith(name_prefix), name
        arrays = port.initial_fields(prog)
        perm_o = port.run(prog, arrays, T)
        assert perm == perm_o
        out = np.empty_like(arrays[0])
        for slot, p in enumerate(perm):
            if out.shape != arrays[p].shape:
                out = np.empty_like(arrays[p])
            plan.download(p, out)
            _equal_chunked(out, arrays[p], f"{name} slot {slot}")
    finally:
        plan.close()


def test_headline_heat3d_so4_1024(port):
    # BASELINE config 5 at N=1 (the driver's headline): 1026^3 + halo, GEO 1 tile, 16 chunks
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 1024, 4, "f32"))
    _big_case(port, prog, 1, "star3d_r2_heat_f32")


def test_headline_wave3d_so8_1024(port):
    # BASELINE config 3: radius 4, 8 z-chunks, the depth-7 ring, 64x24 tile
    prog = hg.build_kernel(hg.KernelSpec("wave", 3, 1024, 8, "f32"))
    _big_case(port, prog, 1, "star3d_r4_wave_f32")


@pytest.mark.parametrize("kind,ext,T", [
    ("wave", [400, 96, 128], 3),   # 3 chunks of 134 planes, ragged last chunk
    ("heat", [300, 64, 64], 3),    # 2 chunks
    ("heat", [520, 40, 72], 2),    # 4 chunks, ragged x (72 = 1 tile + 8)
    ("wave", [700, 24, 200], 2),   # 5 chunks, ragged x/y
])
def test_radius4_multi_chunk(port, kind, ext, T):
    prog = hg.build_kernel(hg.KernelSpec(kind, 3, 8, 8, "f32")).with_extents(ext)
    _big_case(port, prog, T, f"star3d_r4_{kind}_f32")


@pytest.mark.parametrize("ext,T", [([600, 800, 800], 2), ([210, 1000, 900], 1)])
def test_wide_tile_multi_chunk(port, ext, T):
    # the GEO 1 tile with >= 3 z-chunks and the L2 evict_last / evict_first hints
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents(ext)
    _big_case(port, prog, T, "star3d_r2_heat_f32")


def test_field_over_2pow31_elements(port):
    # 1324^3 = 2.32e9 elements per field (> 2^31): 64-bit element indexing in the kernels,
    # the layout, init and transfers
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents([1320] * 3)
    lo, hi = prog.field_bounds(0)
    assert np.prod([b - a for a, b in zip(lo, hi)]) > 2**31
    _big_case(port, prog, 1, "star3d_r2_heat_f32")
