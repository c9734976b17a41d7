# round 2 final 4-GPU pass: whole GPU suite, then the scaling lines (weak/strong, transports,
# deep halos), the simulate path and the reference arm
mkdir -p gpurun_out/final
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/final/tests_4gpu.log 2>&1
echo rc=$? >> gpurun_out/final/tests_4gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo rc=$? >> gpurun_out/final/smoke.log
T(){ n=$1; shift; if [ $n = 1 ]; then python bench.py --gpus 1 "$@"; else python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29520 bench.py --gpus $n "$@"; fi; }
for n in 1 2 4; do timeout 900 bash -c "$(declare -f T); T $n --steps 20 --warmup 5" > gpurun_out/final/weak_n$n.json 2> gpurun_out/final/weak_n$n.err; done
timeout 900 bash -c "$(declare -f T); T 1 --mode strong --steps 5 --warmup 3 --no-e2e" > gpurun_out/final/strong_n1.json 2> gpurun_out/final/strong_n1.err
timeout 900 bash -c "$(declare -f T); T 2 --mode strong --steps 10 --warmup 5 --no-e2e" > gpurun_out/final/strong_n2.json 2> gpurun_out/final/strong_n2.err
for g in 2x2x1 1x2x2 1x1x4 4x1x1 2x1x2 1x4x1; do timeout 900 bash -c "$(declare -f T); T 4 --mode strong --grid $g --steps 10 --warmup 5 --no-e2e" > gpurun_out/final/strong_n4_$g.json 2> gpurun_out/final/strong_n4_$g.err; done
timeout 900 bash -c "$(declare -f T); T 4 --steps 20 --warmup 5 --no-e2e --transport nccl" > gpurun_out/final/weak_n4_nccl.json 2> gpurun_out/final/weak_n4_nccl.err
timeout 900 bash -c "$(declare -f T); T 4 --mode strong --grid 1x2x2 --steps 10 --warmup 5 --no-e2e --transport nccl" > gpurun_out/final/strong_n4_1x2x2_nccl.json 2> gpurun_out/final/strong_n4_1x2x2_nccl.err
timeout 900 bash -c "$(declare -f T); T 4 --steps 20 --warmup 5 --no-e2e --depth 2" > gpurun_out/final/weak_n4_depth2.json 2> gpurun_out/final/weak_n4_depth2.err
timeout 300 python tools/sim_bench.py --gpus 4 --grid 4x1x1 --steps 20 > gpurun_out/final/sim_weak_4x1x1.json 2>&1
timeout 300 python tools/sim_bench.py --gpus 4 --grid 2x2x1 --steps 20 > gpurun_out/final/sim_weak_2x2x1.json 2>&1
timeout 300 python tools/sim_bench.py --gpus 2 --grid 2x1x1 --steps 20 > gpurun_out/final/sim_weak_2x1x1.json 2>&1
timeout 900 python tools/adapter_e2e.py --kind heat --rank 3 --extent 1024 --order 4 --T 100 --calls 2 > gpurun_out/final/adapter_e2e.json 2> gpurun_out/final/adapter_e2e.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final/reference_n1.json 2> gpurun_out/final/reference_n1.err
nvidia-smi topo -m > gpurun_out/final/topo.txt 2>&1
echo done
