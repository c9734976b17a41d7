for v in base d3 d7; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v"
  HG_LIB=$L HG_CHUNKS=0,2,8 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
