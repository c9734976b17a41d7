# round-1 (re-entry) measurements on ONE GPU: gpu tests, bench line of every workload, the
# reference arm, the launch list of the default bench, ncu --set full of the dominant kernels
O=gpurun_out/r1f; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests_1gpu.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
for W in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
  timeout 900 python bench.py --workload $W > $O/bench_$W.log 2>&1; echo "$W rc=$?"
done
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference.log 2>&1; echo "ref rc=$?"
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
python tools/prof_star.py > $O/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o $O/prof_heat3d_so4 python tools/prof_star.py > $O/ncu_heat.log 2>&1; echo "heat rc=$?"
python tools/prof_star.py --kind wave --order 8 > $O/plain_prof2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:starKernel -s 3 -c 1 -o $O/prof_wave3d_so8 python tools/prof_star.py --kind wave --order 8 > $O/ncu_wave.log 2>&1; echo "wave rc=$?"
python tools/prof_resident.py > $O/plain_res.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:residentKernel -s 2 -c 1 -o $O/prof_resident python tools/prof_resident.py > $O/ncu_res.log 2>&1; echo "res rc=$?"
tail -2 $O/gpu_tests_1gpu.log
for f in $O/bench_*.log; do echo "$f: $(tail -1 $f | cut -c1-200)"; done
