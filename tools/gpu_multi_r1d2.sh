O=gpurun_out/r1m; mkdir -p $O
timeout 1800 python -m pytest tests/test_multigpu.py -q > $O/gpu_tests_multigpu_4gpu.log 2>&1; echo "tests rc=$?"
tail -3 $O/gpu_tests_multigpu_4gpu.log
