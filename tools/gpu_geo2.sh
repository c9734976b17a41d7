O=gpurun_out/r1d; mkdir -p $O
HG_STAR_GEO=2 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "serial or medium or config2 or wide or halos or two_step or shallow" > $O/t_geo2.log 2>&1; echo "t rc=$?"
for rep in 1 2; do for g in 1 2; do
  echo -n "geo=$g "; HG_STAR_GEO=$g HG_ONLY=heat3d_so4_1024,heat3d_so4_512,heat3d_so2_1024 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON | tr '\n' ' '; echo
  HG_STAR_GEO=$g python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"  bench heat3d geo=$g\", round(d[\"value\"],1), d[\"clocks\"][\"sm_mhz\"], round(d[\"roofline\"][\"frac\"],3))"
done; done > $O/geo2.log 2>&1
HG_STAR_GEO=2 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:starKernel -s 3 -c 1 python tools/prof_star.py > $O/geo2_ncu.log 2>&1
HG_STAR_GEO=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:starKernel -s 3 -c 1 python tools/prof_star.py >> $O/geo2_ncu.log 2>&1
tail -2 $O/t_geo2.log; cat $O/geo2.log; grep -E "dram__|gpu__time|inst_exec" $O/geo2_ncu.log
