# deep halos on multi-dim grids (sequenced exchange) -- 4 GPUs
mkdir -p gpurun_out/r2_r
timeout 1800 python -m pytest tests/test_multigpu.py -m gpu -q -p no:cacheprovider -k "deep" > gpurun_out/r2_r/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_r/tests.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus 4 --no-e2e"
timeout 600 $B --mode strong --steps 10 --warmup 5 --depth 2 > gpurun_out/r2_r/strong_n4_depth2.json 2> gpurun_out/r2_r/strong_n4_depth2.err
timeout 600 $B --mode strong --steps 10 --warmup 5 > gpurun_out/r2_r/strong_n4.json 2> gpurun_out/r2_r/strong_n4.err
echo done
