"""CPU checks of bench.py's host-side bookkeeping (no GPU): the e2e byte counts follow the
programs (hg_plan_upload_live skips exactly the output slot's store box), the config fields
describe each BASELINE workload, and the reference arm runs on every core it is given."""
import json
import os
import subprocess
import sys

import pytest

import paper_2404_02218_b200 as hg

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402


def test_dead_on_arrival_bytes_follow_the_store_boxes():
    heat = hg.build_kernel(hg.KernelSpec("heat", 3, 64, 4, "f32"))
    assert bench.dead_on_arrival_bytes(heat, 4) == 64 ** 3 * 4      # u_out's core only
    wave = hg.build_kernel(hg.KernelSpec("wave", 3, 40, 8, "f32"))
    assert bench.dead_on_arrival_bytes(wave, 4) == 40 ** 3 * 4      # next's core only
    pw = hg.Program.pw_advection(16, 24, 40)
    assert bench.dead_on_arrival_bytes(pw, 4) == 3 * 16 * 24 * 40 * 4  # su, sv, sw cores


@pytest.mark.parametrize("workload,core,halo", [
    ("heat3d_512", [512, 512, 512], 2), ("wave3d_1024", [1024, 1024, 1024], 4),
    ("pw_advection", [128, 512, 512], 1), ("heat2d_1024", [1024, 1024], 1)])
def test_workload_config_fields(workload, core, halo):
    prog = bench.WORKLOADS[workload]["build"](hg)
    assert bench.core_extents(prog) == core
    assert bench.halo_width(prog) == halo
    assert bench.plan_bytes(prog) > 0


def test_reference_arm_uses_the_given_cores():
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "1", "--ref-planes", "1", "--ref-procs",
                        "2"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["cpu_baseline"]["cores"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0


def test_reference_arm_reports_our_config():
    # the driver compares the two arms' lines: same metric, unit, direction and config
    import argparse
    a = argparse.Namespace(extent=1024, grid=None, mode="weak", workload="heat3d_weak",
                           depth=1, strong_extent=2048)
    c1 = bench.workload_config(a, 1, "p2p")
    assert c1["core_per_gpu"] == [1024, 1024, 1024] and c1["grid"] == [1, 1, 1]
    assert c1["halo"] == 2 and "kernel" not in c1


def test_reference_slab_module_is_config5_planes(ref):
    # the reference arm's sample: the reference's own 1024^3 heat SDO4 module, dim 0 narrowed
    mod = bench._slab_module(ref, 3)
    txt = ref.print(mod)
    assert "[-2,5]x[-2,1026]x[-2,1026]xf32" in txt and "([0,3]x[0,1024]x[0,1024])" in txt
