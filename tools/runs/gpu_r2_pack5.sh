# same-box ncu A/B of the heat 1024^3 star kernel: packed adds (product) vs scalar variant --
# duration, DRAM bytes, L2 hit rate, instructions over launches 3..8, cold (flushed) and warm
mkdir -p gpurun_out/pack5
V=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_scalar.so
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second
for rep in 1 2; do
  ncu --metrics $M --clock-control none -k regex:starKernel -s 2 -c 6 --csv python tools/prof_star.py --steps 8 > gpurun_out/pack5/pack_cold_$rep.csv 2>&1
  HG_LIB=$V ncu --metrics $M --clock-control none -k regex:starKernel -s 2 -c 6 --csv python tools/prof_star.py --steps 8 > gpurun_out/pack5/scalar_cold_$rep.csv 2>&1
  ncu --metrics $M --clock-control none --cache-control none -k regex:starKernel -s 2 -c 6 --csv python tools/prof_star.py --steps 8 > gpurun_out/pack5/pack_warm_$rep.csv 2>&1
  HG_LIB=$V ncu --metrics $M --clock-control none --cache-control none -k regex:starKernel -s 2 -c 6 --csv python tools/prof_star.py --steps 8 > gpurun_out/pack5/scalar_warm_$rep.csv 2>&1
done
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512
for rep in 1 2; do
  python tools/sweep.py > gpurun_out/pack5/sweep_pack_$rep.log 2>&1
  HG_LIB=$V python tools/sweep.py > gpurun_out/pack5/sweep_scalar_$rep.log 2>&1
done
