"""End-to-end GPts/s through the reference-facing drop-in: the reference's
own module (exec::buildKernel, retyped f32) and its own pageable exec::Buffers
(exec::initialFields) go through halogen::exec::gpu::runSerialStencil
(integration/halogen_gpu_adapter.cpp) -- plan creation, uploads from pageable memory through
the pinned staging ring, T steps, downloads back into the Buffers -- exactly what a reference
user gets by swapping exec::runSerialStencil for exec::gpu::runSerialStencil
(tools/halogen.cpp:296-318).  bench.py's `e2e` is the pinned-host path of the C-ABI; this is
the pageable one.  Test infrastructure (uses oracle/_ref to build the reference objects).

  python tools/adapter_e2e.py --kind heat --rank 3 --extent 1024 --order 4 --T 100 --calls 2
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="heat")
    ap.add_argument("--rank", type=int, default=3)
    ap.add_argument("--extent", type=int, default=1024)
    ap.add_argument("--order", type=int, default=4)
    ap.add_argument("--T", type=int, default=100)
    ap.add_argument("--calls", type=int, default=2)
    a = ap.parse_args()
    from oracle import Ref
    ref = Ref()
    L = C.CDLL(os.path.join(REPO, "oracle", "_ref", "libhalogen_gpu_adapter.so"))
    L.hga_run_serial.restype = C.c_void_p
    L.hga_run_serial.argtypes = [C.c_void_p, C.c_void_p, C.c_longlong, C.c_char_p, C.c_int]
    mod = ref.build(a.kind, a.rank, a.extent, a.order, True)
    t0 = time.perf_counter()
    bufs = ref.L.hr_initial_fields(mod)
    t_init = time.perf_counter() - t0
    err = C.create_string_buffer(512)
    out = L.hga_run_serial(mod, bufs, 1, err, 512)  # warm: CUDA context, kernels, staging ring
    assert out, err.value
    ref.L.hr_bufs_free(out)
    times = []
    for _ in range(a.calls):
        t0 = time.perf_counter()
        out = L.hga_run_serial(mod, bufs, a.T, err, 512)
        times.append(time.perf_counter() - t0)
        assert out, err.value
        ref.L.hr_bufs_free(out)
    n = ref.L.hr_bufs_count(bufs)
    nbytes = 0
    for i in range(n):
        eb, rk = C.c_int(), C.c_int()
        shape, lb = (C.c_longlong * 3)(), (C.c_longlong * 3)()
        ref.L.hr_buf_info(bufs, i, C.byref(eb), C.byref(rk), shape, lb)
        m = eb.value
        for d in range(rk.value):
            m *= shape[d]
        nbytes += m
    core = a.extent ** a.rank
    best = min(times)
    print(json.dumps({
        "tool": "adapter_e2e", "path": "halogen::exec::gpu::runSerialStencil (pageable "
        "exec::Buffers, staging ring)", "workload": f"{a.kind}{a.rank}d SDO{a.order} "
        f"{a.extent}^{a.rank} f32", "timesteps_per_call": a.T, "calls": a.calls,
        "seconds_per_call": times, "gpts_per_s": core * a.T / best / 1e9,
        "host_field_bytes": nbytes, "reference_initialFields_s": t_init}), flush=True)


if __name__ == "__main__":
    main()
