# A/B on one box: the round-2 star/apply kernel changes (compile-time ring, per-thread arrives)
# against the library before them (lib/variants/libhalogen_b200_r2base.so), alternating
mkdir -p gpurun_out/ab
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024,pw_advection_128x512x512
for rep in 1 2; do
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_r2base.so python tools/sweep.py > gpurun_out/ab/base_$rep.log 2>&1
  python tools/sweep.py > gpurun_out/ab/new_$rep.log 2>&1
done
bash tools/runs/gpu_r2_prof.sh
