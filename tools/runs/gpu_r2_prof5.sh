# ncu of the shipped kernels after the packed adds (star, resident) and persistent fused-apply
# CTAs: cold single launches (--set full), one warm steady-state launch of the config-5 heat
# kernel (no cache flush, 30 launches in), and the bench launch list
mkdir -p gpurun_out/prof5
NCU="ncu --set full --import-source on --clock-control none"
python tools/prof_star.py --steps 4 > gpurun_out/prof5/plain.log 2>&1 || exit 1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof5/r2_heat3d_so4_1024 python tools/prof_star.py --steps 4 > gpurun_out/prof5/star_heat.log 2>&1
$NCU --cache-control none -k regex:starKernel -s 30 -c 1 -f -o gpurun_out/prof5/r2_heat3d_so4_1024_warm python tools/prof_star.py --steps 32 > gpurun_out/prof5/star_heat_warm.log 2>&1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof5/r2_heat3d_so4_512 python tools/prof_star.py --extent 512 --steps 4 > gpurun_out/prof5/star_512.log 2>&1
$NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof5/r2_wave3d_so8_1024 python tools/prof_star.py --kind wave --order 8 --steps 4 > gpurun_out/prof5/star_wave.log 2>&1
STEPS=4 $NCU -k regex:hg_apply -s 2 -c 1 -f -o gpurun_out/prof5/r2_pw_advection_128x512x512 python tools/prof_pw.py > gpurun_out/prof5/pw.log 2>&1
STEPS=200 $NCU -k regex:residentKernel -s 1 -c 1 -f -o gpurun_out/prof5/r2_resident_heat2d_1024 python tools/prof_resident.py > gpurun_out/prof5/resident.log 2>&1
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof5/bench_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof5/r2_launches_bench_n1.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof5/ncu_bench.log 2>&1
echo done
