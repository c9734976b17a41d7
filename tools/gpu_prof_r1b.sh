# round-1 refresh after the tile-geometry changes: bench lines for every workload, the launch
# list of the default bench, and ncu --set full of the heat and wave star kernels
mkdir -p gpurun_out/r1b
for w in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
  python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/r1b/bench_$w.json 2> gpurun_out/r1b/bench_$w.err
  echo "$w rc=$?"
done
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1b/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1b/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/prof_star.py > gpurun_out/r1b/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/r1b/prof_heat3d_so4 python tools/prof_star.py > gpurun_out/r1b/ncu_heat.log 2>&1; echo "heat rc=$?"
python tools/prof_star.py --kind wave --order 8 > gpurun_out/r1b/plain_prof2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/r1b/prof_wave3d_so8 python tools/prof_star.py --kind wave --order 8 > gpurun_out/r1b/ncu_wave.log 2>&1; echo "wave rc=$?"
