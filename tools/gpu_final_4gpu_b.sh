O=gpurun_out/r1z; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_4gpu_b.log 2>&1; echo "tests rc=$?"
tail -2 $O/gpu_tests_4gpu_b.log
