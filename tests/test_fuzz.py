"""Random stencil modules (tests/randprog.py): the oracle against the reference built from
source (CPU), and every device family against the oracle (GPU).  NaN payloads are compared as
"both NaN" -- IEEE 754 leaves them unspecified (x86 yields 0xffc00000, sm_100a 0x7fffffff)."""
import os
import sys

import numpy as np
import pytest

import paper_2404_02218_b200 as hg
from helpers import fp_hex, prog_to_json
import randprog

HERE = os.path.dirname(os.path.abspath(__file__))
SINGLE = list(range(60))
MULTI = list(range(100, 130))
T = 3


def _texts():
    return [("single", s, randprog.single_apply(s)) for s in SINGLE] + \
           [("multi", s, randprog.multi_apply(s)) for s in MULTI]


@pytest.fixture(scope="module")
def printed(ref):
    """Each random module after the reference's parser + propagate-bounds, and its T-step run."""
    sys.path.insert(0, os.path.join(HERE, "golden"))
    from make_golden import prog_json
    out = []
    L = ref.L
    for kind, seed, text in _texts():
        mod = ref.pipeline(ref.parse(text), "propagate-bounds")
        prog, ops, _ = ref.export_program(mod)
        init = L.hr_initial_fields(mod)
        fin = L.hr_run_serial(mod, L.hr_bufs_clone(init), T)
        assert fin, ref.err()
        fps = ["%016x" % L.hr_fingerprint(fin, i) for i in range(L.hr_bufs_count(fin))]
        out.append((kind, seed, ref.print(mod), prog_json(prog, ops), fps))
    return out


def test_random_modules_reader_and_oracle_match_reference(printed, port):
    for kind, seed, text, pj, fps in printed:
        prog, _, _ = hg.Program.parse(text)
        assert prog_to_json(prog) == pj, (kind, seed)
        arrays = port.initial_fields(prog)
        perm = port.run(prog, arrays, T)
        assert [fp_hex(arrays[p]) for p in perm] == fps, (kind, seed)


def test_random_multi_apply_fusion_on_oracle(printed, port):
    # hg_fuse_applies (temps inlined) == the materialised multi-apply step, on the oracle
    n = 0
    for kind, seed, text, _, fps in printed:
        if kind != "multi":
            continue
        prog, _, _ = hg.Program.parse(text)
        fused = prog.fuse_applies()
        assert fused.prog.napplies == 0
        arrays = port.initial_fields(fused)
        perm = port.run(fused, arrays, T)
        assert [fp_hex(arrays[p]) for p in perm] == fps, seed
        n += 1
    assert n >= 20


def _same(a, b):
    ua = a.view(np.uint32 if a.dtype == np.float32 else np.uint64)
    ub = b.view(np.uint32 if b.dtype == np.float32 else np.uint64)
    return bool(np.all((ua == ub) | (np.isnan(a) & np.isnan(b))))


@pytest.mark.gpu
@pytest.mark.parametrize("family", ["default", "generic", "unfused"])
def test_random_modules_on_gpu(printed, port, monkeypatch, family):
    if family == "generic":
        monkeypatch.setenv("HG_NO_APPLY_JIT", "1")
    if family == "unfused":
        monkeypatch.setenv("HG_NO_FUSE_APPLIES", "1")
    seen = set()
    for kind, seed, text, _, _ in printed:
        prog, _, _ = hg.Program.parse(text)
        plan = hg.Plan(prog)
        plan.init_fields()
        plan.run(T)
        perm, _ = plan.binding()
        got = [plan.download(p) for p in perm]
        seen.add(plan.kernel_name.split("_")[0])
        plan.close()
        arrays = port.initial_fields(prog)
        perm_o = port.run(prog, arrays, T)
        assert perm == perm_o
        for i, (g, o) in enumerate(zip(got, [arrays[p] for p in perm_o])):
            assert _same(g, o), (kind, seed, i, plan.kernel_name)
    assert any(s.startswith("multi") for s in seen)
