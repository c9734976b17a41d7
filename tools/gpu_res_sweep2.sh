mkdir -p gpurun_out/r1d
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or config1 or serial_cases" > gpurun_out/r1d/t_res2.log 2>&1; echo "t rc=$?"; tail -2 gpurun_out/r1d/t_res2.log
for g in 148 128; do for k in 2 4 6 8; do
echo -n "G=$g K=$k "; HG_RES_G=$g HG_RES_K=$k HG_ONLY=heat2d_so2_1024 timeout 120 python tools/sweep.py 2>&1 | grep -v JSON
done; done > gpurun_out/r1d/res_sweep3.log 2>&1
cat gpurun_out/r1d/res_sweep3.log
