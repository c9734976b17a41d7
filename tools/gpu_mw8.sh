O=gpurun_out/r1d; mkdir -p $O
for rep in 1 2; do for v in base mw8; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  for k in 2 3 4; do echo -n "$v K=$k "; HG_LIB=$L HG_RES_K=$k HG_ONLY=heat2d_so2_1024 timeout 120 python tools/sweep.py 2>&1 | grep -v JSON; done
done; done > $O/mw8.log 2>&1
cat $O/mw8.log
