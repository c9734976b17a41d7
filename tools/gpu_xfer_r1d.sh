mkdir -p gpurun_out/r1d
timeout 300 python tools/xfer_probe.py > gpurun_out/r1d/xfer2.log 2>&1; echo "xfer rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host_transfers or host_api" > gpurun_out/r1d/t_xfer.log 2>&1; echo "t rc=$?"
timeout 900 python bench.py --steps 100 > gpurun_out/r1d/bench2.log 2>&1; echo "bench rc=$?"
cat gpurun_out/r1d/xfer2.log; tail -3 gpurun_out/r1d/t_xfer.log; tail -1 gpurun_out/r1d/bench2.log
