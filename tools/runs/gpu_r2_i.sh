# round 2: pitch rule + geometry rule verification (parity + bench lines + 17-line neighbours)
mkdir -p gpurun_out/r2_i
timeout 1200 python -m pytest tests/test_bench_shapes.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_i/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_i/tests.log
for w in heat3d_weak heat3d_512 wave3d_1024; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_i/n1_$w.json 2> gpurun_out/r2_i/n1_$w.err
done
python - > gpurun_out/r2_i/lines.log 2>&1 <<'PY'
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2404_02218_b200 as hg
s = torch.cuda.current_stream(); sh = ctypes.c_void_p(s.cuda_stream)
for x in (1566, 1598, 1630, 2108, 2140, 2172, 1024):
    prog = hg.build_kernel(hg.KernelSpec("heat", 3, 8, 4, "f32")).with_extents([1024, 1024, x])
    plan = hg.Plan(prog); plan.init_fields(stream=sh); plan.run(6, stream=sh)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(s); plan.run(12, stream=sh); e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 12
    print(x, "pitch", plan.layout(0).pitch, "lines", plan.layout(0).pitch // 32, f"{prog.core_points() / ms / 1e6:.1f} GPts/s", flush=True)
    plan.close()
PY
echo done
