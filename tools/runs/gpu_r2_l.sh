# round 2: shipped 10-slot 128x12 ring -- parity, N=1 bench lines, ncu of the shipped kernels
mkdir -p gpurun_out/r2_l gpurun_out/prof3
timeout 1500 python -m pytest tests/test_bench_shapes.py tests/test_gpu_parity.py tests/test_fuzz.py tests/test_adapter.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_l/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_l/tests.log
for w in heat3d_weak heat3d_512 wave3d_1024 pw_advection; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_l/n1_$w.json 2> gpurun_out/r2_l/n1_$w.err
done
timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 > gpurun_out/r2_l/n1_heat2d_1024.json 2> gpurun_out/r2_l/n1_heat2d_1024.err
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof3/r2_heat3d_so4_1024 python tools/prof_star.py --steps 4 > gpurun_out/prof3/star_heat.log 2>&1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof3/r2_heat3d_so4_512 python tools/prof_star.py --extent 512 --steps 4 > gpurun_out/prof3/star_512.log 2>&1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof3/r2_wave3d_so8_1024 python tools/prof_star.py --kind wave --order 8 --steps 4 > gpurun_out/prof3/star_wave.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof3/r2_launches_bench_n1.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof3/ncu_bench.log 2>&1
echo done
