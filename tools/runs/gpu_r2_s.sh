mkdir -p gpurun_out/r2_s
timeout 1800 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "deep or nccl" > gpurun_out/r2_s/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_s/tests.log
echo done
