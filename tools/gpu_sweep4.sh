for c in 1 2 4 8; do
  echo "=== cluster $c"
  HG_CLUSTER=$c HG_ONLY=heat3d_so4_1024,wave3d_so8_1024,heat3d_so4_512 HG_CHUNKS=3,8,16,24 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
for c in 1 4 8; do
python tools/prof_star.py --chunks 16 > /dev/null 2>&1 && \
HG_CLUSTER=$c ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py --chunks 16 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/cluster=$c /"
done
HG_CLUSTER=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
