timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024 HG_CHUNKS=0,1,2,4,8,16,32 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
for c in 1 4 16; do
python tools/prof_star.py --chunks $c > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py --chunks $c 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/chunks=$c /"
done
