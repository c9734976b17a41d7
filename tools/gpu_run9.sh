for V in "" "HG_FUSE_SCRATCH=1"; do
env $V HG_DMP_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 200 --warmup 5 --no-e2e > gpurun_out/b2q.log 2>&1; echo "[$V] $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b2q.log)"; grep "steps 200" gpurun_out/b2q.log
done
