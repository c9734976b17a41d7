for v in base t32; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v"
  HG_LIB=$L HG_ONLY=wave3d_so8_1024,heat3d_so8_1024,heat3d_so4_1024 HG_CHUNKS=0,4,8 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
  HG_LIB=$L timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "serial or medium" 2>&1 | tail -1
done
