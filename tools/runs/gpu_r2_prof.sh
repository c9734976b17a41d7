# round 2 ncu captures of the shipped kernels (one GPU; each program exits 0 without ncu first)
mkdir -p gpurun_out/prof
NCU="ncu --set full --import-source on --clock-control none"
python tools/prof_star.py --steps 4 && $NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof/r2_star_heat3d_so4_1024 python tools/prof_star.py --steps 4 > gpurun_out/prof/star_heat.log 2>&1
python tools/prof_star.py --kind wave --order 8 --steps 4 && $NCU -k regex:starKernel -s 2 -c 1 -f -o gpurun_out/prof/r2_star_wave3d_so8_1024 python tools/prof_star.py --kind wave --order 8 --steps 4 > gpurun_out/prof/star_wave.log 2>&1
python tools/prof_pw.py && $NCU -k regex:hg_apply -s 1 -c 1 -f -o gpurun_out/prof/r2_pw_advection_128x512x512 python tools/prof_pw.py > gpurun_out/prof/pw.log 2>&1
STEPS=200 python tools/prof_resident.py && STEPS=200 $NCU -k regex:residentKernel -s 1 -c 1 -f -o gpurun_out/prof/r2_resident_heat2d_1024 python tools/prof_resident.py > gpurun_out/prof/resident.log 2>&1
python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/bench_plain.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/r2_launches_bench_n1.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/prof/ncu_bench.log 2>&1
echo done
