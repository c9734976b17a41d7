free -g > gpurun_out/r2_box.txt; nproc >> gpurun_out/r2_box.txt; nvidia-smi topo -m >> gpurun_out/r2_box.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=25 > gpurun_out/r2_gpu_tests_a.log 2>&1
echo rc=$? >> gpurun_out/r2_gpu_tests_a.log
