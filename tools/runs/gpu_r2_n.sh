# multi-GPU A/B: 10-slot (shipped) vs 8-slot ring, same 4-GPU box, alternating
mkdir -p gpurun_out/r2_n
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29530 bench.py --gpus 4 --no-e2e"
R8=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_ring8.so
for rep in 1 2; do
  for g in 4x1x1 2x2x1; do
    timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 > gpurun_out/r2_n/ship_strong_${g}_$rep.json 2>/dev/null
    HG_LIB=$R8 timeout 600 $B --mode strong --grid $g --steps 10 --warmup 5 > gpurun_out/r2_n/ring8_strong_${g}_$rep.json 2>/dev/null
  done
  HG_DMP_PROFILE=1 timeout 600 $B --mode strong --grid 4x1x1 --steps 10 --warmup 5 > gpurun_out/r2_n/prof_strong_4x1x1_$rep.json 2> gpurun_out/r2_n/prof_strong_4x1x1_$rep.err
done
echo done
