python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/prof_star.py > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/prof_r1_heat3d_so4 python tools/prof_star.py > gpurun_out/ncu_heat.log 2>&1; echo "heat rc=$?"
python tools/prof_star.py --kind wave --order 8 > gpurun_out/plain_prof2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/prof_r1_wave3d_so8 python tools/prof_star.py --kind wave --order 8 > gpurun_out/ncu_wave.log 2>&1; echo "wave rc=$?"
