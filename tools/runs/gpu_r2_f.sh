# round 2: packed standalone puts (x faces) + receiver slab unpack; resident 2D changes
mkdir -p gpurun_out/r2_bench_f
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r2_bench_f/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_bench_f/tests.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2"
for g in 2x1x1 1x1x2; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench_f/strong_n2_$g.json 2> gpurun_out/r2_bench_f/strong_n2_$g.err
done
HG_DMP_PROFILE=1 timeout 600 $B --mode strong --grid 1x1x2 --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench_f/strong_n2_1x1x2_prof.json 2> gpurun_out/r2_bench_f/strong_n2_1x1x2_prof.err
timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench_f/n1_heat2d.json 2> gpurun_out/r2_bench_f/n1_heat2d.err
HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_r2base.so timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_f/n1_heat2d_base.json 2> gpurun_out/r2_bench_f/n1_heat2d_base.err
echo done
