O=gpurun_out/r1z; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_4gpu_c.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_c.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_n1_c.log 2>&1; echo "n1 rc=$?"
tail -2 $O/gpu_tests_4gpu_c.log; tail -1 $O/bench_n1_c.log | cut -c1-200
