"""Multi-process halo swap over NVLink (one rank per GPU, CUDA IPC peer memory): bitwise
against the oracle, halos included.  Needs >= 2 GPUs; the CPU side of the rank protocol is
covered by tests/test_dist_gloo.py."""
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--kind", "heat", "--rank", "3", "--extent", "48", "--order", "4", "--T", "6"],
    ["--kind", "wave", "--rank", "3", "--extent", "40", "--order", "8", "--T", "5"],
    ["--kind", "heat", "--rank", "2", "--extent", "64", "--order", "2", "--T", "7"],
    ["--kind", "wave", "--rank", "3", "--extent", "64", "--order", "4", "--T", "9",
     "--calls", "1,3,5"],
    ["--kind", "heat", "--rank", "3", "--extent", "100", "--order", "8", "--T", "6",
     "--calls", "4,2"],
    # bench.py's e2e path: pinned host fields, live uploads over poisoned buffers, then runs
    ["--kind", "heat", "--rank", "3", "--extent", "48", "--order", "4", "--T", "5",
     "--calls", "2,3", "--upload"],
    ["--kind", "wave", "--rank", "3", "--extent", "40", "--order", "8", "--T", "4",
     "--upload"],
])
def test_ipc_dmp_two_ranks(args):
    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    for nproc, grid in ((2, None), (min(n, 4), "2x2x1" if "3" == args[3] else "2x2"),
                        (min(n, 4), "1x2x2" if "3" == args[3] else "1x4"),
                        (min(n, 4), "4x1x1" if "3" == args[3] else "4x1")):
        if nproc < 4 and grid:
            continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone",
               "--nproc-per-node", str(nproc), os.path.join(REPO, "tools", "dmp_check.py")] + args
        if grid:
            cmd += ["--grid", grid]
        r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("args", [
    ["--kind", "heat", "--rank", "3", "--extent", "48", "--order", "4", "--T", "5"],
    ["--kind", "wave", "--rank", "3", "--extent", "40", "--order", "8", "--T", "4",
     "--calls", "1,3"],
])
def test_nccl_transport_baseline(args):
    # the NCCL transport (C++: pack, ncclSend/ncclRecv on a side stream, unpack, interior
    # units overlapped) is bit-exact too, halos included
    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    for nproc, grid in ((2, "2x1x1"), (2, "1x1x2"), (4, "2x2x1"), (4, "1x2x2")):
        if nproc > n:
            continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone",
               "--nproc-per-node", str(nproc), os.path.join(REPO, "tools", "dmp_check.py"),
               "--transport", "nccl", "--grid", grid] + args
        r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("geo", ["1", "3"])
@pytest.mark.parametrize("grid", ["2x1x1", "1x2x2", "2x2x1"])
def test_ipc_dmp_wide_tile(grid, geo):
    # the wide star tiles (forced) with the fused next-step swap over NVLink
    n = _ngpus()
    nproc = int(np.prod([int(x) for x in grid.split("x")]))
    if n < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
           str(nproc), os.path.join(REPO, "tools", "dmp_check.py"), "--kind", "heat", "--rank",
           "3", "--extent", "64", "--order", "4", "--T", "6", "--calls", "2,4", "--grid", grid]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, HG_STAR_GEO=geo))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name,grids", [("indep2f_2d", ["2x1", "1x2", "2x2"]),
                                        ("twin3_3d_f64", ["2x1x1", "1x1x2", "2x2x1"])])
def test_ipc_dmp_multi_apply(name, grids):
    # a step of several applies: one swap per load, every swapped field over NVLink
    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    for grid in grids:
        nproc = int(np.prod([int(x) for x in grid.split("x")]))
        if nproc > n:
            continue
        cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone",
               "--nproc-per-node", str(nproc), os.path.join(REPO, "tools", "dmp_check.py"),
               "--golden", name, "--grid", grid, "--T", "5", "--calls", "2,3"]
        r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("spec,grid,T", [
    (("wave", 3, 24, 8), [3, 1, 1], 4), (("heat", 3, 24, 4), [2, 2, 1], 4),
    (("heat", 2, 24, 2), [2, 2], 3),
])
def test_simulate_ranks_spread_over_devices(port, spec, grid, T):
    # one process, ranks round-robin over the visible GPUs: peer pointers + cross-device events
    import numpy as np
    import paper_2404_02218_b200 as hg
    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    init = hg.initial_fields(prog)
    nr = int(np.prod(grid))
    out = hg.simulate(prog, grid, init, T, devices=[r % n for r in range(nr)])
    arrays = [b.data.copy() for b in init]
    perm = port.run(prog, arrays, T)
    for b, p in zip(out, perm):
        assert np.array_equal(b.data.view(np.uint32), arrays[p].view(np.uint32))


@pytest.mark.gpu
@pytest.mark.parametrize("kind,order,extents,grid,T,calls", [
    # heat SDO4, local 256x64x64 per rank: 4 z-chunks -> boundary_last reorder + per-chunk
    # fused-put completion counters on the z faces
    ("heat", 4, "512x64x64", "2x1x1", 5, "2,3"),
    ("heat", 4, "512x128x64", "2x2x1", 4, None),
    # wave SDO8, local 400x48x48: 3 chunks, radius 4, the 3-cycle rotation
    ("wave", 8, "800x48x48", "2x1x1", 4, "1,3"),
    # the wide 128x12 tile (planes >= 768^2) with 3 chunks per rank: the bench's kernel
    ("heat", 4, "400x800x800", "2x1x1", 3, None),
    ("heat", 4, "400x800x800", "4x1x1", 3, None),
    ("heat", 4, "512x256x128", "1x2x2", 3, None),
])
def test_ipc_dmp_multi_chunk(kind, order, extents, grid, T, calls):
    # the per-rank shapes of the weak/strong bench (many z-chunks per
    # rank) under the oracle's restatement of RankHooks::swap, halos included
    n = _ngpus()
    nproc = int(np.prod([int(x) for x in grid.split("x")]))
    if n < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
           str(nproc), os.path.join(REPO, "tools", "dmp_check.py"), "--kind", kind, "--rank",
           "3", "--order", str(order), "--extents", extents, "--grid", grid, "--T", str(T)]
    if calls:
        cmd += ["--calls", calls]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("kind,rank,order,extents,grid,T,calls,extra", [
    # grids that split the contiguous last dim: x faces travel as packed slabs [y][z][w],
    # sent by the producing CTAs in 16-byte stores and unpacked by the receiving CTAs' producer
    # warp before their TMA loads (and by the stand-alone put on a call's first step)
    ("heat", 3, 4, "256x128x512", "1x1x2", 5, "1,4", []),
    ("heat", 3, 4, "200x800x1600", "1x1x2", 3, None, []),          # wide 128x12 tile
    ("wave", 3, 8, "400x48x192", "1x1x2", 4, "2,2", []),
    ("heat", 3, 8, "120x40x250", "1x1x2", 3, None, []),            # ragged, 125 = odd width
    ("heat", 2, 2, "256x512", "1x2", 6, "3,3", []),
    ("heat", 3, 4, "256x128x512", "1x1x2", 4, "2,2", ["--upload"]),
    ("heat", 3, 4, "192x256x256", "1x2x2", 4, None, []),
    ("heat", 3, 4, "256x256x256", "2x1x2", 3, "1,2", []),
    ("wave", 3, 8, "200x96x200", "1x1x4", 3, None, []),
])
def test_ipc_dmp_x_faces(kind, rank, order, extents, grid, T, calls, extra):
    n = _ngpus()
    nproc = int(np.prod([int(x) for x in grid.split("x")]))
    if n < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
           str(nproc), os.path.join(REPO, "tools", "dmp_check.py"), "--kind", kind, "--rank",
           str(rank), "--order", str(order), "--extents", extents, "--grid", grid, "--T",
           str(T)] + extra
    if calls:
        cmd += ["--calls", calls]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("spec,grid,T", [
    (("heat", 3, 48, 4), [2, 1, 1], 5), (("heat", 3, 48, 4), [1, 1, 2], 5),
    (("wave", 3, 40, 8), [1, 2, 1], 4), (("heat", 2, 64, 2), [1, 2], 6),
    (("heat", 3, 64, 4), [2, 2, 1], 4), (("heat", 3, 64, 4), [1, 2, 2], 3),
])
def test_simulate_one_rank_per_device(port, spec, grid, T):
    # hg_sim_run with one rank per GPU takes the multi-process protocol (fused NVLink swap,
    # in-kernel flag waits, packed x faces) from one host thread: gathered result == serial
    import paper_2404_02218_b200 as hg
    n = _ngpus()
    nr = int(np.prod(grid))
    if n < nr:
        pytest.skip(f"needs {nr} GPUs")
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    init = hg.initial_fields(prog)
    out = hg.simulate(prog, grid, init, T, devices=list(range(nr)))
    arrays = [b.data.copy() for b in init]
    perm = port.run(prog, arrays, T)
    for b, p in zip(out, perm):
        assert np.array_equal(b.data.view(np.uint32), arrays[p].view(np.uint32))


@pytest.mark.gpu
def test_stuck_peer_reports_instead_of_hanging():
    # a neighbour that never runs: rank 0's halo wait times out and surfaces as HG_ETRAP
    # ("... did not arrive for epoch e within 2.0 s ...") instead of a hung GPU
    n = _ngpus()
    if n < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
           os.path.join(REPO, "tools", "stuck_peer.py")]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "STUCK-PEER REPORTED" in r.stdout, r.stdout[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("kind,rank,order,extents,grid,T,calls,depth,transport", [
    # deep halos (communication-avoiding): depth*h-wide halos exchanged
    # every `depth` steps, the ring recomputed redundantly; odd call lengths end a round early
    ("heat", 3, 4, "256x96x128", "2x1x1", 7, "3,4", 2, "p2p"),
    ("heat", 3, 4, "256x96x256", "1x1x2", 6, "2,4", 2, "p2p"),     # packed x, extended region
    ("wave", 3, 8, "400x48x96", "2x1x1", 7, "5,2", 2, "p2p"),
    ("heat", 3, 2, "300x64x64", "2x1x1", 8, "8", 3, "p2p"),
    ("heat", 2, 2, "512x256", "2x1", 9, "4,5", 3, "p2p"),
    ("heat", 3, 4, "200x800x800", "2x1x1", 5, None, 2, "p2p"),     # wide tile, 1024-like planes
    ("heat", 3, 4, "256x96x128", "2x1x1", 7, "3,4", 2, "nccl"),
    ("wave", 3, 8, "200x96x192", "1x1x2", 5, None, 2, "nccl"),
    ("heat", 3, 4, "192x256x128", "1x2x1", 6, "1,5", 2, "p2p"),     # y split
    ("heat", 3, 4, "400x64x96", "4x1x1", 7, "3,4", 2, "p2p"),
    # several split dims: the sequenced (dim-ordered, corner-carrying) round exchange
    ("heat", 3, 4, "192x128x256", "2x2x1", 6, "1,5", 2, "p2p"),
    ("heat", 3, 4, "192x128x256", "1x2x2", 7, None, 2, "p2p"),
    ("heat", 3, 2, "120x96x160", "2x1x2", 7, "4,3", 3, "p2p"),
    ("wave", 3, 8, "160x96x96", "2x2x1", 5, "2,3", 2, "p2p"),
    ("heat", 2, 2, "256x256", "2x2", 9, "4,5", 3, "p2p"),
    ("heat", 3, 4, "192x128x256", "2x2x1", 6, "1,5", 2, "nccl"),   # NCCL, dim-ordered stages
    ("wave", 3, 8, "160x96x96", "1x2x2", 5, None, 2, "nccl"),
])
def test_ipc_dmp_deep_halo(kind, rank, order, extents, grid, T, calls, depth, transport):
    n = _ngpus()
    nproc = int(np.prod([int(x) for x in grid.split("x")]))
    if n < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node",
           str(nproc), os.path.join(REPO, "tools", "dmp_check.py"), "--kind", kind, "--rank",
           str(rank), "--order", str(order), "--extents", extents, "--grid", grid, "--T",
           str(T), "--depth", str(depth), "--transport", transport]
    if calls:
        cmd += ["--calls", calls]
    r = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("spec,grid,T,depth", [
    (("heat", 3, 48, 4), [2, 1, 1], 7, 2), (("wave", 3, 48, 8), [1, 1, 2], 5, 2),
    (("heat", 3, 64, 2), [1, 4, 1], 7, 3), (("heat", 3, 64, 2), [2, 2, 1], 7, 3),
    (("heat", 3, 48, 4), [1, 2, 2], 5, 2),
])
def test_simulate_deep_halo(port, spec, grid, T, depth):
    # simulate with deep halos (one rank per GPU): gathered cores == the serial run
    import paper_2404_02218_b200 as hg
    n = _ngpus()
    nr = int(np.prod(grid))
    if n < nr:
        pytest.skip(f"needs {nr} GPUs")
    prog = hg.build_kernel(hg.KernelSpec(*spec, "f32"))
    init = hg.initial_fields(prog)
    out = hg.simulate(prog, grid, init, T, devices=list(range(nr)), depth=depth)
    arrays = [b.data.copy() for b in init]
    perm = port.run(prog, arrays, T)
    for b, p in zip(out, perm):
        assert np.array_equal(b.data.view(np.uint32), arrays[p].view(np.uint32))
