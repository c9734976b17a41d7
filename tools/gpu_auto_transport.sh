O=gpurun_out/r1m; mkdir -p $O
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29583 bench.py --gpus 4 --steps 50 --mode strong --grid 1x1x4 --no-e2e > $O/bench_auto_1x1x4.log 2>&1; echo "auto 1x1x4 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29584 bench.py --gpus 4 > $O/bench_auto_weak4.log 2>&1; echo "auto weak rc=$?"
for f in $O/bench_auto_*.log; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value'],1), d['config']['transport'], (d.get('e2e') or {}).get('value'))"; done
