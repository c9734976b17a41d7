mkdir -p gpurun_out/r1d
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or config1 or serial_cases" > gpurun_out/r1d/t_res.log 2>&1; echo "t rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1d/smoke2.log 2>&1; echo "smoke rc=$?"
HG_ONLY=heat2d_so2_1024 timeout 300 python tools/sweep.py > gpurun_out/r1d/res_sweep.log 2>&1
HG_NO_RESIDENT=1 HG_ONLY=heat2d_so2_1024 timeout 300 python tools/sweep.py >> gpurun_out/r1d/res_sweep.log 2>&1
timeout 600 python bench.py --workload heat2d_1024 --steps 2000 > gpurun_out/r1d/bench_h2d.log 2>&1; echo "bench rc=$?"
tail -15 gpurun_out/r1d/t_res.log; cat gpurun_out/r1d/smoke2.log gpurun_out/r1d/res_sweep.log | grep -v JSON; tail -1 gpurun_out/r1d/bench_h2d.log | cut -c1-600
