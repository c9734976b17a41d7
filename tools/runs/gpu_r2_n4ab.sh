# weak N=4 (4x1x1), fused P2P vs C++ NCCL transport, alternating, 200 timed steps; P2P phase times
mkdir -p gpurun_out/n4ab
T(){ python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 "$@"; }
for rep in 1 2; do
  timeout 300 bash -c "$(declare -f T); T --steps 200 --warmup 5 --no-e2e --no-cpu-baseline" > gpurun_out/n4ab/p2p_$rep.json 2> gpurun_out/n4ab/p2p_$rep.err
  timeout 300 bash -c "$(declare -f T); T --steps 200 --warmup 5 --no-e2e --no-cpu-baseline --transport nccl" > gpurun_out/n4ab/nccl_$rep.json 2> gpurun_out/n4ab/nccl_$rep.err
done
HG_DMP_PROFILE=1 timeout 300 bash -c "$(declare -f T); T --steps 50 --warmup 5 --no-e2e --no-cpu-baseline" > gpurun_out/n4ab/p2p_prof.json 2> gpurun_out/n4ab/p2p_prof.err
