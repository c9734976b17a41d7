"""hgrun: the CLI counterpart of the reference's `halogen run-serial / simulate --check /
bench` (proj/tools/halogen.cpp) on the GPU path, fed with the reference's own printed
modules (tests/golden/)."""
import os
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HGRUN = os.path.join(REPO, "paper_2404_02218_b200", "bin", "hgrun")


def _run(args, stdin=None):
    return subprocess.run([HGRUN] + args, input=stdin, capture_output=True, text=True,
                          timeout=300)


def test_hgrun_built_and_usage():
    assert os.access(HGRUN, os.X_OK)
    r = _run([])
    assert r.returncode == 2 and "usage" in r.stderr


def test_hgrun_parse_errors_are_reported():
    r = _run(["run-serial", "-"], stdin="not a module")
    assert r.returncode == 1 and "<xir>:1:1" in r.stderr


@pytest.mark.gpu
def test_hgrun_run_serial_matches_reference(golden, tmp_path):
    done = 0
    for c in golden["serial"] + golden["authored"]:
        if not c.get("text") or c["T"] > 20:
            continue
        f = tmp_path / "m.xir"
        f.write_text(c["text"])
        r = _run(["run-serial", str(f), "-t", str(c["T"])])
        assert r.returncode == 0, r.stderr
        fps = [ln.split()[2] for ln in r.stdout.splitlines() if ln.startswith("field ")]
        assert fps == [h.lstrip("0") or "0" for h in c["final_fp"]], c.get("name", c.get("spec"))
        done += 1
    assert done >= 23


@pytest.mark.gpu
def test_hgrun_simulate_check(golden, tmp_path):
    for c in golden["decomposed"] + golden["decomposed_authored"]:
        f = tmp_path / "d.xir"
        f.write_text(c["text"])
        r = _run(["simulate", str(f), "-t", str(c["T"]), "--check"])
        assert r.returncode == 0, r.stderr + r.stdout
        fps = [ln.split()[2] for ln in r.stdout.splitlines() if ln.startswith("field ")]
        assert fps == [h.lstrip("0") or "0" for h in c["sim_fp"]]
        assert r.stdout.count("bitwise match") == len(c["sim_fp"])


@pytest.mark.gpu
def test_hgrun_bench_csv():
    r = _run(["bench", "--kind", "heat", "--rank", "3", "--extent", "128", "--order", "4",
              "-t", "20"])
    assert r.returncode == 0, r.stderr
    hdr, row = r.stdout.strip().splitlines()
    assert hdr == "label,core_points,steps,seconds,gpts_per_s"
    label, pts, steps, secs, gpts = row.split(",")
    assert label == "heat-3d-n128-o4" and int(pts) == 128 ** 3 and int(steps) == 20
    assert float(gpts) > 0
    r = _run(["bench", "--kind", "wave", "--rank", "3", "--extent", "64", "--order", "8",
              "-t", "5", "--grid", "2x1x1"])
    assert r.returncode == 0, r.stderr
    assert r.stdout.splitlines()[1].startswith("wave-3d-n64-o8-g2x1x1,")
