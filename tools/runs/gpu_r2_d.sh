# round 2: CT-ring star kernel, per-thread arrives, CTA-wide x unpack, deep-halo bands
timeout 1800 python -m pytest tests/test_bench_shapes.py tests/test_gpu_parity.py tests/test_multigpu.py tests/test_fuzz.py -m gpu -q -x -p no:cacheprovider --durations=10 > gpurun_out/r2_gpu_tests_d.log 2>&1
echo rc=$? >> gpurun_out/r2_gpu_tests_d.log
mkdir -p gpurun_out/r2_bench_d
for w in heat3d_weak wave3d_1024 pw_advection heat3d_512 heat2d_1024; do
  timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_d/n1_$w.json 2> gpurun_out/r2_bench_d/n1_$w.err
done
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2"
timeout 600 $B --steps 20 --warmup 5 --no-e2e > gpurun_out/r2_bench_d/weak_n2.json 2> gpurun_out/r2_bench_d/weak_n2.err
for g in 2x1x1 1x1x2 1x2x1; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench_d/strong_n2_$g.json 2> gpurun_out/r2_bench_d/strong_n2_$g.err
done
timeout 600 $B --mode strong --grid 1x1x2 --steps 10 --warmup 5 --no-e2e --transport nccl > gpurun_out/r2_bench_d/strong_n2_1x1x2_nccl.json 2> gpurun_out/r2_bench_d/strong_n2_1x1x2_nccl.err
echo done
