O=gpurun_out/r1u; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "live_upload or zero_steps" > $O/t1.log 2>&1; echo "t1 rc=$?"; tail -1 $O/t1.log
timeout 1500 python -m pytest tests/test_multigpu.py -q -k "two_ranks" > $O/t2.log 2>&1; echo "t2 rc=$?"; tail -1 $O/t2.log
