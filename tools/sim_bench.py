"""GPts/s of hg_sim_run -- the stepping loop behind halogen::exec::gpu::simulate (the drop-in of
exec::simulate, simulator.cpp:1066-1203) -- with one rank per GPU in ONE process, for
comparison with bench.py's torchrun line on the same grid.

  python tools/sim_bench.py --gpus 4 --grid 2x2x1 --extent 1024 --steps 20

Weak scaling shape (BASELINE config 5): extent^3 core per rank.  Fields are initialised on the
device (the reference's initValue at each rank's origin = scatterRank of the global init).
The timed region is the hg_sim_run call (it returns after every rank finished, so host time
around it is the step time), after a warm-up call.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import paper_2404_02218_b200 as hg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--grid", default=None)
    ap.add_argument("--extent", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--depth", type=int, default=1)
    a = ap.parse_args()
    grid = [int(x) for x in a.grid.split("x")] if a.grid else [a.gpus, 1, 1]
    n = grid[0] * grid[1] * grid[2]
    E = a.extent
    glob = hg.build_kernel(hg.KernelSpec("heat", 3, E, 4, "f32")).with_extents(
        [E * grid[0], E * grid[1], E * grid[2]])
    local, dc = glob.decompose(grid, depth=a.depth)
    plans, dmps = [], []
    for r in range(n):
        pl = hg.Plan(local, r % a.gpus)
        c = hg.coord_from_rank(r, grid)
        pl.init_fields(origin=[c[d] * dc.core[d] for d in range(3)])
        plans.append(pl)
        dmps.append(hg.Dmp(pl, dc, r, depth=a.depth))
    arr = (C.c_void_p * n)(*[d.h for d in dmps])
    hg.check(hg.lib().hg_sim_connect(arr, n))
    hg.check(hg.lib().hg_sim_run(arr, n, a.warmup, None))
    t0 = time.perf_counter()
    hg.check(hg.lib().hg_sim_run(arr, n, a.steps, None))
    secs = time.perf_counter() - t0
    pts = local.core_points() * n * a.steps
    print(json.dumps({"tool": "sim_bench", "path": "hg_sim_run (simulate drop-in)",
                      "grid": grid, "gpus": a.gpus, "core_per_rank": list(dc.core[:3]),
                      "depth": a.depth, "steps": a.steps, "ms_per_step": secs / a.steps * 1e3,
                      "gpts_per_s": pts / secs / 1e9, "kernel": plans[0].kernel_name}),
          flush=True)
    for d in dmps:
        d.close()
    for p in plans:
        p.close()


if __name__ == "__main__":
    main()
