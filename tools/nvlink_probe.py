"""NVLink evidence for the fused swap: two ranks of one process on two
GPUs (hg_sim_run, the fused protocol), heat SDO4 with 512^3 per rank split along z (2x1x1) or
x (1x1x2: packed slabs).  Run under ncu on ONE device:

  ncu --devices 0 -k regex:starKernel -s 3 -c 1 --metrics nvltx__bytes.sum,nvlrx__bytes.sum,\
gpu__time_duration.sum python tools/nvlink_probe.py --grid 2x1x1

The profiled launch is a middle step (fused send of the next step's halo); the expected payload
is printed for comparison (the send box of one face: 2 planes / 2 columns of the core).
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2404_02218_b200 as hg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="2x1x1")
    ap.add_argument("--extent", type=int, default=512)
    ap.add_argument("--steps", type=int, default=6)
    a = ap.parse_args()
    grid = [int(x) for x in a.grid.split("x")]
    E = a.extent
    glob = hg.build_kernel(hg.KernelSpec("heat", 3, E, 4, "f32")).with_extents(
        [E * grid[0], E * grid[1], E * grid[2]])
    local, dc = glob.decompose(grid)
    plans, dmps = [], []
    for r in range(2):
        pl = hg.Plan(local, r)
        c = hg.coord_from_rank(r, grid)
        pl.init_fields(origin=[c[d] * dc.core[d] for d in range(3)])
        plans.append(pl)
        dmps.append(hg.Dmp(pl, dc, r, timeout_s=120.0))
    arr = (C.c_void_p * 2)(*[d.h for d in dmps])
    hg.check(hg.lib().hg_sim_connect(arr, 2))
    hg.check(hg.lib().hg_sim_run(arr, 2, a.steps, None))
    face = E * E * 2 * 4  # one face's send box: 2 planes (z) or 2 columns (x) of E^2, f32
    print(f"grid {grid}: payload per fused send (one face) = {face} bytes; "
          f"bytes put by rank 0 over {a.steps} steps = {dmps[0].bytes_exchanged()}", flush=True)
    for d in dmps:
        d.close()
    for p in plans:
        p.close()


if __name__ == "__main__":
    main()
