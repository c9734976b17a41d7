timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu4.log
for N in 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 400 --warmup 5 > gpurun_out/bench_n$N.log 2>&1; echo "bench$N rc=$?"; tail -1 gpurun_out/bench_n$N.log | cut -c1-330; grep -o '"e2e": {[^}]*}' gpurun_out/bench_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --mode strong > gpurun_out/bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"; tail -1 gpurun_out/bench_strong_n$N.log | cut -c1-330
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 2 --steps 400 --warmup 5 --no-e2e > gpurun_out/bench_n2b.log 2>&1; echo "bench2 rc=$?"; tail -1 gpurun_out/bench_n2b.log | cut -c1-330
timeout 300 python bench.py --steps 400 > gpurun_out/bench_n1b.log 2>&1; echo "bench1 rc=$?"; tail -1 gpurun_out/bench_n1b.log
timeout 300 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
