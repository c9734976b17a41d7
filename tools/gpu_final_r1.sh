# round-1 final measurements: bench lines (every workload; weak/strong 1-4 GPUs; reference arm)
# then the launch list and ncu --set full of the dominant kernels (single-process commands)
bash tools/gpu_bench_r1c.sh
mkdir -p gpurun_out/r1b
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1b/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r1b/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/prof_star.py > gpurun_out/r1b/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/r1b/prof_heat3d_so4 python tools/prof_star.py > gpurun_out/r1b/ncu_heat.log 2>&1; echo "heat rc=$?"
python tools/prof_star.py --kind wave --order 8 > gpurun_out/r1b/plain_prof2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o gpurun_out/r1b/prof_wave3d_so8 python tools/prof_star.py --kind wave --order 8 > gpurun_out/r1b/ncu_wave.log 2>&1; echo "wave rc=$?"
