# re-entry check: full gpu test suite, smoke, default bench line
mkdir -p gpurun_out/r1d
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r1d/gpu_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1d/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r1d/bench.log 2>&1; echo "bench rc=$?"
tail -2 gpurun_out/r1d/gpu_tests.log; tail -1 gpurun_out/r1d/bench.log
