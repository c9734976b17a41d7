O=gpurun_out/r1m; mkdir -p $O
for g in 1x1x4 1x2x2 2x2x1; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 50 --no-e2e --mode strong --grid $g --transport nccl > $O/bench_strong_n4_nccl_$g.log 2>&1; echo "$g rc=$?"
tail -1 $O/bench_strong_n4_nccl_$g.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nccl $g', round(d['value'],1), round(d['ms_per_step'],3), d['clocks']['sm_mhz'])"
done
