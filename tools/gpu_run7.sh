timeout 300 python bench.py --steps 400 --no-e2e --no-cpu-baseline > gpurun_out/b1.log 2>&1; echo "n1 $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b1.log) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/b1.log)"
for F in 0 1; do
if [ $F = 1 ]; then export HG_NOFUSE=1; else unset HG_NOFUSE; fi
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$F bench.py --gpus 2 --steps 400 --warmup 5 --no-e2e > gpurun_out/b2_$F.log 2>&1; echo "n2 nofuse=$F $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/b2_$F.log) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/b2_$F.log) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/b2_$F.log)"
done
