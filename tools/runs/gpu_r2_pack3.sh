# The product library with packed adds in both families: single-GPU parity suites, the PW A/B
# (persistent x packed), and the bench lines of configs 2-5.
mkdir -p gpurun_out/pack3
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_bench_shapes.py tests/test_fuzz.py tests/test_adapter.py -m gpu -x -q > gpurun_out/pack3/tests.log 2>&1; echo rc=$? >> gpurun_out/pack3/tests.log
python tools/pw_ab.py 3 > gpurun_out/pack3/pw_ab.log 2>&1
for w in pw_advection heat3d_512 wave3d_1024; do
  timeout 600 python bench.py --workload $w > gpurun_out/pack3/n1_$w.json 2> gpurun_out/pack3/n1_$w.err
done
timeout 600 python bench.py > gpurun_out/pack3/weak_n1.json 2> gpurun_out/pack3/weak_n1.err
HG_JIT_PACK=0 timeout 600 python bench.py --workload pw_advection --no-cpu-baseline --no-e2e > gpurun_out/pack3/n1_pw_nopack.json 2>/dev/null
timeout 600 python bench.py --workload pw_advection --no-cpu-baseline --no-e2e > gpurun_out/pack3/n1_pw_pack2.json 2>/dev/null
