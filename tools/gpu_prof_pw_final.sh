O=gpurun_out/r1p; mkdir -p $O
python bench.py --workload pw_advection --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_pw.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hg_apply -s 3 -c 1 -o $O/prof_pw_apply python bench.py --workload pw_advection --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_pw.log 2>&1; echo "ncu pw rc=$?"
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/prof_star.py > $O/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o $O/prof_heat3d_so4 python tools/prof_star.py > $O/ncu_heat.log 2>&1; echo "heat rc=$?"
