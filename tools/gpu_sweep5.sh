for o in 0 1 2; do
  echo "=== order $o"
  HG_ORDER=$o HG_ONLY=heat3d_so4_1024,wave3d_so8_1024,heat3d_so4_512 HG_CHUNKS=3,8,16,32 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
for o in 0 1 2; do
python tools/prof_star.py --chunks 16 > /dev/null 2>&1 && \
HG_ORDER=$o ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py --chunks 16 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/order=$o /"
done
HG_ORDER=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
