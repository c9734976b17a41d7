# round 2: 10-slot compile-time ring on the 128x12 tile, re-tested with the 35-line pitch
mkdir -p gpurun_out/r2_k
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512
for rep in 1 2; do
  python tools/sweep.py > gpurun_out/r2_k/ship_$rep.log 2>&1
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_geo1ct.so python tools/sweep.py > gpurun_out/r2_k/ct_$rep.log 2>&1
done
for d in 1 2 3 4; do HG_JIT_DEPTH=$d HG_ONLY=pw_advection_128x512x512 python tools/sweep.py > gpurun_out/r2_k/pw_depth$d.log 2>&1; done
echo done
