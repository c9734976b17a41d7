# round 2: producer-side x unpack (batches ahead of the TMA loads)
mkdir -p gpurun_out/r2_j
timeout 1500 python -m pytest tests/test_multigpu.py -m gpu -q -x -p no:cacheprovider -k "x_faces or deep or multi_chunk or one_rank_per_device or nccl" > gpurun_out/r2_j/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_j/tests.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 2"
for g in 2x1x1 1x1x2 1x2x1; do
  timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 --no-e2e > gpurun_out/r2_j/strong_n2_$g.json 2> gpurun_out/r2_j/strong_n2_$g.err
done
echo done
