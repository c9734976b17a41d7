# round-1 bench lines (default K/W) for every workload + weak/strong scaling on 4 GPUs
mkdir -p gpurun_out/r1c
for W in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
timeout 600 python bench.py --workload $W > gpurun_out/r1c/r1_bench_$W.log 2>&1; echo "$W rc=$?"
done
for N in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > gpurun_out/r1c/r1_bench_weak_n$N.log 2>&1; echo "weak$N rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --steps 100 --no-e2e --mode strong > gpurun_out/r1c/r1_bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"
done
timeout 900 python bench.py --steps 50 --no-e2e --no-cpu-baseline --mode strong > gpurun_out/r1c/r1_bench_strong_n1.log 2>&1; echo "strong1 rc=$?"
timeout 600 python bench.py --impl reference > gpurun_out/r1c/r1_bench_reference.log 2>&1; echo "ref rc=$?"
