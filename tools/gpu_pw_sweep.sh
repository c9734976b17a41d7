mkdir -p gpurun_out/r1d
for rep in 1 2; do
HG_ONLY=pw_advection_128x512x512 HG_CHUNKS=0,1,2,3,4,5,6,7,8,12,16 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON
done > gpurun_out/r1d/pw_sweep.log 2>&1
for d in 3 4 5 6; do echo "depth $d"; HG_JIT_DEPTH=$d HG_ONLY=pw_advection_128x512x512 HG_CHUNKS=0,4,8 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON; done >> gpurun_out/r1d/pw_sweep.log 2>&1
cat gpurun_out/r1d/pw_sweep.log
