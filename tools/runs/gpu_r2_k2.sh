mkdir -p gpurun_out/r2_k2
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv > gpurun_out/r2_k2/smi.txt
for rep in 1 2 3; do
  python tools/sweep.py > gpurun_out/r2_k2/ship_$rep.log 2>&1
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_geo1ct.so python tools/sweep.py > gpurun_out/r2_k2/ct_$rep.log 2>&1
done
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit,temperature.gpu --format=csv >> gpurun_out/r2_k2/smi.txt
echo done
