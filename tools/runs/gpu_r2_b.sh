# round 2: new dmp (packed x faces, unit order, bounded waits, C++ NCCL transport, sim fused path)
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py tests/test_adapter.py -m gpu -q -x -p no:cacheprovider --durations=15 > gpurun_out/r2_gpu_tests_b.log 2>&1
echo rc=$? >> gpurun_out/r2_gpu_tests_b.log
