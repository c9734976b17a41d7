O=gpurun_out/r1d; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or config1 or serial_cases" > $O/t_res3.log 2>&1; echo "t rc=$?"
for rep in 1 2; do for k in 1 2 4; do echo -n "K=$k "; HG_RES_K=$k HG_ONLY=heat2d_so2_1024 timeout 120 python tools/sweep.py 2>&1 | grep -v JSON; done; done > $O/res_final.log 2>&1
cat $O/res_final.log; tail -1 $O/t_res3.log
