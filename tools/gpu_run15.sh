for W in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
timeout 600 python bench.py --workload $W > gpurun_out/r1_bench_$W.log 2>&1; echo "$W rc=$?"
done
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/r1_bench_weak_n$N.log 2>&1; echo "weak$N rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --steps 100 --no-e2e --mode strong > gpurun_out/r1_bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"
done
timeout 900 python bench.py --steps 50 --no-e2e --no-cpu-baseline --mode strong > gpurun_out/r1_bench_strong_n1.log 2>&1; echo "strong1 rc=$?"
python bench.py --workload pw_advection --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:hg_apply -s 3 -c 1 -o gpurun_out/prof_r1_pw_apply python bench.py --workload pw_advection --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pw.log 2>&1; echo "ncu pw rc=$?"
