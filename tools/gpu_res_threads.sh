O=gpurun_out/r1d; mkdir -p $O
for rep in 1 2; do for v in base res768 res1024; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  for k in 2 4; do echo -n "$v K=$k "; HG_LIB=$L HG_RES_K=$k HG_ONLY=heat2d_so2_1024 timeout 120 python tools/sweep.py 2>&1 | grep -v JSON; done
done; done > $O/res_threads.log 2>&1
HG_LIB=paper_2404_02218_b200/lib/variants/libhalogen_b200_res1024.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or config1" > $O/t_res1024.log 2>&1; echo "t rc=$?"
cat $O/res_threads.log; tail -1 $O/t_res1024.log
