mkdir -p gpurun_out/r1d
timeout 300 python tools/xfer_probe.py > gpurun_out/r1d/xfer3.log 2>&1; echo "xfer rc=$?"
HG_XFER=ce timeout 300 python tools/xfer_probe.py > gpurun_out/r1d/xfer3_ce.log 2>&1; echo "xfer ce rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "host_transfers or host_api" > gpurun_out/r1d/t_xfer2.log 2>&1; echo "t rc=$?"
timeout 900 python bench.py --steps 100 > gpurun_out/r1d/bench3.log 2>&1; echo "bench rc=$?"
cat gpurun_out/r1d/xfer3.log gpurun_out/r1d/xfer3_ce.log; tail -3 gpurun_out/r1d/t_xfer2.log; tail -1 gpurun_out/r1d/bench3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e'])"
