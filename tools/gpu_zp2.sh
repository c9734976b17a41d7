O=gpurun_out/r1d; mkdir -p $O
L2=paper_2404_02218_b200/lib/variants/libhalogen_b200_zp2.so
HG_LIB=$L2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "serial or medium or config or wide or two_step or transfers or zero_steps or split" > $O/t_zp2.log 2>&1; echo "t rc=$?"; tail -1 $O/t_zp2.log
for rep in 1 2; do for v in base zp2 zp2d7; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== $v rep $rep"
  HG_LIB=$L HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
  HG_LIB=$L python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"bench heat3d\", round(d[\"value\"],1), d[\"clocks\"][\"sm_mhz\"])"
done; done > $O/zp2.log 2>&1
cat $O/zp2.log
