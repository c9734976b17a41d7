# round 2: resident B checks, final 1-GPU profiles of the shipped kernels, N=1 bench lines,
# adapter e2e (pageable Buffers through halogen::exec::gpu::runSerialStencil)
mkdir -p gpurun_out/r2_h gpurun_out/prof2
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_adapter.py tests/test_cli.py -m gpu -q -x -p no:cacheprovider -k "resident or config1 or heat or dropin or run_serial" > gpurun_out/r2_h/tests_resident.log 2>&1
echo rc=$? >> gpurun_out/r2_h/tests_resident.log
for w in heat3d_weak wave3d_1024 pw_advection heat3d_512; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_h/n1_$w.json 2> gpurun_out/r2_h/n1_$w.err
done
timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 > gpurun_out/r2_h/n1_heat2d_1024.json 2> gpurun_out/r2_h/n1_heat2d_1024.err
timeout 900 python tools/adapter_e2e.py --kind heat --rank 3 --extent 1024 --order 4 --T 100 --calls 2 > gpurun_out/r2_h/adapter_e2e_heat3d_1024.json 2> gpurun_out/r2_h/adapter_e2e.err
NCU="ncu --set full --import-source on --clock-control none"
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof2/r2_heat3d_so4_1024 python tools/prof_star.py --steps 4 > gpurun_out/prof2/star_heat.log 2>&1
STEPS=200 $NCU -k regex:residentKernel -s 1 -c 1 -f -o gpurun_out/prof2/r2_resident_heat2d_1024 python tools/prof_resident.py > gpurun_out/prof2/resident.log 2>&1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof2/r2_heat3d_so4_512 python tools/prof_star.py --extent 512 --steps 4 > gpurun_out/prof2/star_512.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof2/r2_launches_bench_n1.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof2/ncu_bench.log 2>&1
echo done
