"""The reference-side drop-in (integration/halogen_gpu_adapter.cpp): the reference's own
modules and Buffers go through halogen::exec::gpu::runSerialStencil / simulate on the B200 and
come back bitwise equal to the reference's CPU executors run on the same inputs in the same
process (oracle/_ref, built from /root/reference; the built .so files travel to the GPU box)."""
import ctypes as C
import os

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ADAPTER = os.path.join(REPO, "oracle", "_ref", "libhalogen_gpu_adapter.so")


@pytest.fixture(scope="module")
def adapter(ref):
    if not os.path.exists(ADAPTER):
        pytest.skip("adapter not built (make -C oracle adapter)")
    L = C.CDLL(ADAPTER)
    for n in ("hga_run_serial", "hga_simulate"):
        f = getattr(L, n)
        f.restype = C.c_void_p
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_char_p, C.c_int]
    L.hga_lowered_recognised.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
    return L


@pytest.mark.parametrize("spec,grid", [(("heat", 2, 12, 2), "2x2"), (("wave", 3, 24, 8), "3x1x1"),
                                       (("heat", 3, 32, 4), "2x2x2"), (("wave", 1, 16, 4), "4")])
def test_lowered_module_recognised(ref, adapter, spec, grid):
    # the `halogen bench --grid` module (tools/halogen.cpp:320-323) maps back to its dmp level
    mod = ref.build(*spec, True)
    err = C.create_string_buffer(300)
    low = ref.pipeline(mod, f"propagate-bounds,decompose grid={grid},lower-dmp-to-mpi")
    assert adapter.hga_lowered_recognised(low, err, 300) == 1, err.value
    # also after the reference interpreter has run it (value slots get numbered lazily)
    init = ref.L.hr_initial_fields(mod)
    assert ref.L.hr_simulate(low, init, 2, 0)
    assert adapter.hga_lowered_recognised(low, err, 300) == 1, err.value
    dmp = ref.pipeline(mod, f"propagate-bounds,decompose grid={grid}")
    assert adapter.hga_lowered_recognised(dmp, err, 300) == 0


def test_adapter_loads_and_exports(adapter):
    assert hasattr(adapter, "hga_run_serial") and hasattr(adapter, "hga_simulate")


def _fps(ref, bufs):
    return [ref.L.hr_fingerprint(bufs, i) for i in range(ref.L.hr_bufs_count(bufs))]


@pytest.mark.gpu
@pytest.mark.parametrize("spec,T", [
    (("heat", 2, 1024, 2), 100), (("heat", 3, 64, 4), 5), (("wave", 3, 48, 8), 4),
    (("heat", 3, 40, 8), 3), (("wave", 2, 90, 4), 6), (("heat", 1, 50, 4), 3),
    (("copy", 3, 12, 2), 2),
])
@pytest.mark.parametrize("f32", [1, 0])
def test_run_serial_stencil_dropin(ref, adapter, spec, T, f32):
    if spec[2] >= 1024 and not f32:
        pytest.skip("config-1 shape is an f32 case")
    mod = ref.build(*spec, bool(f32))
    init = ref.L.hr_initial_fields(mod)
    cpu = ref.L.hr_run_serial(mod, ref.L.hr_bufs_clone(init), T)
    err = C.create_string_buffer(512)
    gpu = adapter.hga_run_serial(mod, ref.L.hr_bufs_clone(init), T, err, 512)
    assert gpu, err.value.decode()
    assert _fps(ref, gpu) == _fps(ref, cpu)


@pytest.mark.gpu
@pytest.mark.parametrize("spec,grid,T", [
    (("heat", 2, 12, 2), "2x2", 3), (("wave", 1, 16, 4), "4", 4), (("copy", 2, 8, 2), "2x1", 2),
    (("heat", 3, 32, 4), "2x2x2", 3), (("wave", 3, 24, 8), "3x1x1", 4),
    (("heat", 3, 48, 2), "1x2x3", 2),
])
def test_simulate_dropin(ref, adapter, spec, grid, T):
    mod = ref.build(*spec, True)
    dmod = ref.pipeline(mod, "propagate-bounds,decompose grid=" + grid)
    init = ref.L.hr_initial_fields(mod)
    cpu = ref.L.hr_simulate(dmod, init, T, 0)
    assert cpu, ref.err()
    err = C.create_string_buffer(512)
    gpu = adapter.hga_simulate(dmod, init, T, err, 512)
    assert gpu, err.value.decode()
    assert _fps(ref, gpu) == _fps(ref, cpu)


@pytest.mark.gpu
@pytest.mark.parametrize("spec,grid,T", [
    (("heat", 2, 12, 2), "2x2", 3), (("heat", 3, 32, 4), "2x2x2", 2),
    (("wave", 3, 24, 8), "3x1x1", 3),
])
def test_simulate_lowered_mpi_module(ref, adapter, spec, grid, T):
    # the exact module `halogen bench --grid` times: propagate-bounds,decompose,lower-dmp-to-mpi
    mod = ref.build(*spec, True)
    low = ref.pipeline(mod, "propagate-bounds,decompose grid=" + grid + ",lower-dmp-to-mpi")
    init = ref.L.hr_initial_fields(mod)
    cpu = ref.L.hr_simulate(low, init, T, 0)
    assert cpu, ref.err()
    err = C.create_string_buffer(512)
    gpu = adapter.hga_simulate(low, init, T, err, 512)
    assert gpu, err.value.decode()
    assert _fps(ref, gpu) == _fps(ref, cpu)


@pytest.mark.gpu
def test_multi_apply_dropin(ref, adapter, golden):
    # multi-apply modules (chained and independent applies) through the drop-in: serial runs
    # and decomposed simulate, bitwise against the reference's executors in-process
    n = 0
    for c in golden["authored"]:
        if "applies" not in c["program"]:
            continue
        mod = ref.parse(c["text"])
        init = ref.L.hr_initial_fields(mod)
        cpu = ref.L.hr_run_serial(mod, ref.L.hr_bufs_clone(init), c["T"])
        err = C.create_string_buffer(512)
        gpu = adapter.hga_run_serial(mod, ref.L.hr_bufs_clone(init), c["T"], err, 512)
        assert gpu, err.value.decode()
        assert _fps(ref, gpu) == _fps(ref, cpu), c["name"]
        n += 1
    for c in golden["decomposed_authored"]:
        mod = ref.parse(c["global_text"])
        dmod = ref.parse(c["text"])
        init = ref.L.hr_initial_fields(mod)
        cpu = ref.L.hr_simulate(dmod, init, c["T"], 0)
        err = C.create_string_buffer(512)
        gpu = adapter.hga_simulate(dmod, init, c["T"], err, 512)
        assert gpu, err.value.decode()
        assert _fps(ref, gpu) == _fps(ref, cpu), c["name"]
        n += 1
    assert n >= 5


def test_adapter_errors_like_the_reference(ref, adapter):
    # wrong field count -> TrapError text (serial.cpp:68-69 analogue), never a crash
    mod = ref.build("heat", 2, 8, 2, True)
    init = ref.L.hr_initial_fields(mod)
    empty = ref.L.hr_bufs_clone(init)
    # a module with no all-field function
    bad = ref.parse("builtin.module {\n}\n")
    err = C.create_string_buffer(512)
    assert not adapter.hga_run_serial(bad, empty, 1, err, 512)
    assert b"step function" in err.value
