O=gpurun_out/r1d; mkdir -p $O
timeout 300 python tools/xfer_probe.py > $O/xfer4.log 2>&1; echo "xfer rc=$?"
HG_NO_STAGING=1 timeout 300 python tools/xfer_probe.py > $O/xfer4_nostage.log 2>&1; echo "xfer ns rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_adapter.py -x -q -k "pageable or host_transfers or host_api or adapter" > $O/t_stage.log 2>&1; echo "t rc=$?"
grep -E "plan|flat" $O/xfer4.log; echo; grep pageable $O/xfer4_nostage.log; tail -2 $O/t_stage.log
