# round 2: sanitizers (2 GPUs), A/B of the GEO1 ring revert, x-split strong N=2 after the flat put
mkdir -p gpurun_out/ab2 gpurun_out/r2_bench_e
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024
for rep in 1 2; do
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_r2base.so python tools/sweep.py > gpurun_out/ab2/base_$rep.log 2>&1
  python tools/sweep.py > gpurun_out/ab2/new_$rep.log 2>&1
done
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2"
for g in 2x1x1 1x1x2; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench_e/strong_n2_$g.json 2> gpurun_out/r2_bench_e/strong_n2_$g.err
done
HG_DMP_PROFILE=1 timeout 600 $B --mode strong --grid 1x1x2 --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_bench_e/strong_n2_1x1x2_prof.json 2> gpurun_out/r2_bench_e/strong_n2_1x1x2_prof.err
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x -p no:cacheprovider -k "x_faces or deep or stuck" > gpurun_out/r2_bench_e/tests_x.log 2>&1
bash tools/runs/gpu_r2_sanitize.sh
echo done
