mkdir -p gpurun_out/r1d
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "shallow or authored" > gpurun_out/r1d/t_shallow.log 2>&1; echo "shallow rc=$?"
REPS=30 timeout 600 python tools/debug_flux_unfused.py > gpurun_out/r1d/dbg3.log 2>&1; echo "dbg rc=$?"
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r1d/gpu_tests2.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/r1d/t_shallow.log; cat gpurun_out/r1d/dbg3.log | tail -3; tail -5 gpurun_out/r1d/gpu_tests2.log
