O=gpurun_out/r1fb; mkdir -p $O
for W in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
  timeout 900 python bench.py --workload $W > $O/bench_$W.log 2>&1; echo "$W rc=$?"
done
python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "launch rc=$?"
for f in $O/bench_*.log; do echo "$f: $(tail -1 $f | cut -c1-120)"; done
