# round 2, 4 GPUs: full GPU suite + multi-GPU measurements (packed x faces, NCCL C++, deep halos, sim)
set -x
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/r2_gpu_tests_4gpu.log 2>&1
echo rc=$? >> gpurun_out/r2_gpu_tests_4gpu.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4"
mkdir -p gpurun_out/r2_bench
timeout 600 $B --steps 20 --warmup 5 > gpurun_out/r2_bench/weak_n4.json 2> gpurun_out/r2_bench/weak_n4.err
timeout 600 $B --steps 20 --warmup 5 --no-e2e --depth 2 > gpurun_out/r2_bench/weak_n4_depth2.json 2> gpurun_out/r2_bench/weak_n4_depth2.err
for g in 2x2x1 1x2x2 1x1x4 4x1x1; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench/strong_n4_$g.json 2> gpurun_out/r2_bench/strong_n4_$g.err
done
for g in 2x2x1 1x1x4; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e --transport nccl > gpurun_out/r2_bench/strong_n4_${g}_nccl.json 2> gpurun_out/r2_bench/strong_n4_${g}_nccl.err
done
timeout 600 $B --steps 20 --warmup 5 --no-e2e --transport nccl > gpurun_out/r2_bench/weak_n4_nccl.json 2> gpurun_out/r2_bench/weak_n4_nccl.err
timeout 300 python tools/sim_bench.py --gpus 4 --grid 4x1x1 --steps 20 > gpurun_out/r2_bench/sim_weak_4x1x1.json 2>&1
timeout 300 python tools/sim_bench.py --gpus 4 --grid 2x2x1 --steps 20 > gpurun_out/r2_bench/sim_weak_2x2x1.json 2>&1
timeout 300 python tools/sim_bench.py --gpus 4 --grid 2x2x1 --steps 20 --depth 2 > gpurun_out/r2_bench/sim_weak_2x2x1_depth2.json 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench/n1.json 2> gpurun_out/r2_bench/n1.err
echo done
