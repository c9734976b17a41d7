timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for N in 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 400 --warmup 5 --no-e2e > gpurun_out/bench_n$N.log 2>&1; echo "bench$N rc=$?"; tail -1 gpurun_out/bench_n$N.log | cut -c1-400
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --mode strong > gpurun_out/bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"; tail -1 gpurun_out/bench_strong_n$N.log | cut -c1-400
done
timeout 300 python bench.py --steps 400 --no-e2e > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/bench_n1.log
timeout 600 python bench.py --steps 50 --no-e2e --no-cpu-baseline --mode strong > gpurun_out/bench_strong_n1.log 2>&1; echo "strong1 rc=$?"; tail -1 gpurun_out/bench_strong_n1.log | cut -c1-400
