O=gpurun_out/r1d; mkdir -p $O
for rep in 1 2; do
for v in hint nohint; do
  if [ $v = hint ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v rep $rep"
  HG_LIB=$L HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024,heat3d_so8_1024 HG_CHUNKS=0 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
  HG_LIB=$L python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"bench heat3d\", round(d[\"value\"],1), d[\"clocks\"])"
done
done > $O/hint.log 2>&1
for v in hint nohint; do
  if [ $v = hint ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  HG_LIB=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 3 -c 2 python tools/prof_star.py > $O/hint_ncu_$v.log 2>&1
  HG_LIB=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 3 -c 2 python tools/prof_star.py --kind wave --order 8 >> $O/hint_ncu_$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "serial or medium or wide or config or shape" > $O/t_hint.log 2>&1; echo "t rc=$?"
cat $O/hint.log; grep -E "dram__|gpu__time" $O/hint_ncu_*.log; tail -2 $O/t_hint.log
