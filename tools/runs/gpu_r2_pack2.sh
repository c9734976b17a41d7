# A/B on one box: packed adds (HG_PACK=2 variant) against the product star kernels.
# Parity of the variant first (star instances incl. the benched shapes), then burst (sweep.py)
# and sustained (bench.py, 400 timed steps) rates, alternating.
mkdir -p gpurun_out/pack2
V=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_p2.so
HG_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_bench_shapes.py -m gpu -x -q > gpurun_out/pack2/tests_p2.log 2>&1; echo rc=$? >> gpurun_out/pack2/tests_p2.log
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024
for rep in 1 2 3; do
  python tools/sweep.py > gpurun_out/pack2/base_$rep.log 2>&1
  HG_LIB=$V python tools/sweep.py > gpurun_out/pack2/p2_$rep.log 2>&1
done
for rep in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pack2/bench_base_$rep.json 2>/dev/null
  HG_LIB=$V timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/pack2/bench_p2_$rep.json 2>/dev/null
  timeout 600 python bench.py --workload wave3d_1024 --no-cpu-baseline --no-e2e > gpurun_out/pack2/bench_wave_base_$rep.json 2>/dev/null
  HG_LIB=$V timeout 600 python bench.py --workload wave3d_1024 --no-cpu-baseline --no-e2e > gpurun_out/pack2/bench_wave_p2_$rep.json 2>/dev/null
done
