for rep in 1 2; do
for v in base oldwave w32y15d7; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v rep $rep"
  HG_LIB=$L HG_ONLY=wave3d_so8_1024,heat3d_so8_1024 HG_CHUNKS=0 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
done
python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
