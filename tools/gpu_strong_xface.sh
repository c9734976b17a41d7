O=gpurun_out/r1m; mkdir -p $O
for g in 2x2x1 1x2x2 4x1x1 1x1x4; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 100 --no-e2e --mode strong --grid $g > $O/bench_strong_n4_$g.log 2>&1; echo "$g rc=$?"
tail -1 $O/bench_strong_n4_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$g', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
