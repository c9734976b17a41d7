for v in base x32y8 x8y32; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v"
  HG_LIB=$L HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024 HG_CHUNKS=0,8,16,24 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
  python tools/prof_star.py > /dev/null 2>&1 && HG_LIB=$L ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py 2>&1 | grep -E "dram__|gpu__time"
  HG_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "serial or medium" 2>&1 | tail -1
done
