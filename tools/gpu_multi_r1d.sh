# multi-GPU: the full gpu suite on 4 GPUs (runs the 2/4-rank tests), weak + strong bench lines
O=gpurun_out/r1m; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q > $O/gpu_tests_4gpu.log 2>&1; echo "tests rc=$?"
for N in 2 4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N bench.py --gpus $N > $O/bench_weak_n$N.log 2>&1; echo "weak$N rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2956$N bench.py --gpus $N --steps 100 --no-e2e --mode strong > $O/bench_strong_n$N.log 2>&1; echo "strong$N rc=$?"
done
timeout 900 python bench.py --steps 50 --no-e2e --no-cpu-baseline --mode strong > $O/bench_strong_n1.log 2>&1; echo "strong1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --impl reference --steps 10 --warmup 3 > $O/bench_reference_n4.log 2>&1; echo "ref4 rc=$?"
tail -2 $O/gpu_tests_4gpu.log
for f in $O/bench_*.log; do echo "$f: $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d.get('ms_per_step'), (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1)"; done
