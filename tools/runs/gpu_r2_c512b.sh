# wave-aware auto chunking (single-GPU plain steps): 1-GPU parity suites, smoke, then config 2
# auto (now 12 chunks) vs the old default (8), alternating, and the config 5 line (unchanged: 16)
mkdir -p gpurun_out/c512b
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_bench_shapes.py tests/test_fuzz.py tests/test_adapter.py -m gpu -x -q > gpurun_out/c512b/tests.log 2>&1; echo rc=$? >> gpurun_out/c512b/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/c512b/smoke.log 2>&1; echo rc=$? >> gpurun_out/c512b/smoke.log
for rep in 1 2; do
  timeout 300 python bench.py --workload heat3d_512 --no-cpu-baseline --no-e2e > gpurun_out/c512b/auto_$rep.json 2>/dev/null
  timeout 300 python bench.py --workload heat3d_512 --chunks 8 --no-cpu-baseline --no-e2e > gpurun_out/c512b/c8_$rep.json 2>/dev/null
done
timeout 300 python bench.py --workload heat3d_512 > gpurun_out/c512b/n1_heat3d_512.json 2>/dev/null
