# packed-add heat 1024^3: z-chunk count (16 = auto, 64 planes) vs shorter chunks, back to back
# (steady state, power-capped) and the DRAM bytes per launch under ncu
mkdir -p gpurun_out/pack6
export HG_ONLY=heat3d_so4_1024
for rep in 1 2 3; do
  HG_CHUNKS=16,20,24,32 python tools/sweep.py > gpurun_out/pack6/sweep_$rep.log 2>&1
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in 16 24 32; do
  ncu --metrics $M --clock-control none -k regex:starKernel -s 2 -c 3 --csv python tools/prof_star.py --steps 6 --chunks $c > gpurun_out/pack6/ncu_c$c.csv 2>&1
done
