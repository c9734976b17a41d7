timeout 1200 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -15 gpurun_out/pytest_mgpu.log
for N in 4 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 400 --warmup 5 --no-e2e > gpurun_out/bench_n$N.log 2>&1; echo "bench$N rc=$?"; tail -1 gpurun_out/bench_n$N.log | cut -c1-330
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --mode strong > gpurun_out/bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"; tail -1 gpurun_out/bench_strong_n$N.log | cut -c1-330
done
