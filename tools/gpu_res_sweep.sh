mkdir -p gpurun_out/r1d
for g in 148 128 96 64; do for k in 1 2 4 6 8; do
echo -n "G=$g K=$k "; HG_RES_G=$g HG_RES_K=$k HG_ONLY=heat2d_so2_1024 timeout 120 python tools/sweep.py 2>&1 | grep -v JSON
done; done > gpurun_out/r1d/res_sweep2.log 2>&1
cat gpurun_out/r1d/res_sweep2.log
