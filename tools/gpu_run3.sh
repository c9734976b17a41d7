nvidia-smi topo -m | head -5
timeout 900 python -m pytest tests/test_multigpu.py -q -x > gpurun_out/pytest_mgpu.log 2>&1; echo "mgpu rc=$?"; tail -30 gpurun_out/pytest_mgpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/bench_n2.log 2>&1; echo "bench2 rc=$?"; tail -4 gpurun_out/bench_n2.log
timeout 300 python bench.py --steps 400 --no-e2e --no-cpu-baseline > gpurun_out/bench_n1.log 2>&1; echo "bench1 rc=$?"; tail -2 gpurun_out/bench_n1.log
