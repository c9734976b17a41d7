O=gpurun_out/r1d; mkdir -p $O
for rep in 1 2; do HG_ONLY=heat3d_so4_512,heat3d_so4_1024 HG_CHUNKS=0,4,6,7,8,12,14,16,24 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON; done > $O/h512_chunks.log 2>&1
HG_ONLY=wave3d_so8_1024 HG_CHUNKS=0,4,6,8,10,12 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON >> $O/h512_chunks.log 2>&1
cat $O/h512_chunks.log
