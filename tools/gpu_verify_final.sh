O=gpurun_out/r1v; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests_1gpu.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --workload heat2d_1024 > $O/bench_heat2d_1024.log 2>&1; echo "h2d rc=$?"
timeout 600 python bench.py > $O/bench_default.log 2>&1; echo "bench rc=$?"
tail -2 $O/gpu_tests_1gpu.log; cat $O/smoke.log; tail -1 $O/bench_heat2d_1024.log | cut -c1-300; tail -1 $O/bench_default.log | cut -c1-300
