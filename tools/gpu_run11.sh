timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
HG_ONLY=pw_advection_128x512x512 HG_CHUNKS=0,1,2,4 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
HG_ONLY=pw_advection_128x512x512 HG_NO_APPLY_JIT=1 HG_CHUNKS=0 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
