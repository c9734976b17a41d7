# round 2 closing 4-GPU pass after packed adds / persistent fused-apply / rows-per-thread: the whole GPU suite under HG_DEBUG_GUARDS (parity + out-of-bounds
# canaries), smoke, then the bench lines (N=1 every workload, weak N=2/4, strong, transports,
# deep halos, simulate drop-in, adapter e2e, reference arm)
mkdir -p gpurun_out/final6
HG_DEBUG_GUARDS=1 timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/final6/tests_4gpu_guards.log 2>&1
echo rc=$? >> gpurun_out/final6/tests_4gpu_guards.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final6/smoke.log 2>&1; echo rc=$? >> gpurun_out/final6/smoke.log
T(){ n=$1; shift; if [ $n = 1 ]; then python bench.py --gpus 1 "$@"; else python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29550 bench.py --gpus $n "$@"; fi; }
for n in 1 2 4; do timeout 900 bash -c "$(declare -f T); T $n --steps 20 --warmup 5" > gpurun_out/final6/weak_n$n.json 2> gpurun_out/final6/weak_n$n.err; done
for w in heat3d_512 wave3d_1024 pw_advection; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/final6/n1_$w.json 2> gpurun_out/final6/n1_$w.err; done
timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 > gpurun_out/final6/n1_heat2d_1024.json 2> gpurun_out/final6/n1_heat2d_1024.err
timeout 900 bash -c "$(declare -f T); T 1 --mode strong --steps 5 --warmup 3 --no-e2e" > gpurun_out/final6/strong_n1.json 2> gpurun_out/final6/strong_n1.err
timeout 900 bash -c "$(declare -f T); T 2 --mode strong --steps 10 --warmup 5 --no-e2e" > gpurun_out/final6/strong_n2.json 2> gpurun_out/final6/strong_n2.err
for g in 2x2x1 1x2x2 1x1x4; do timeout 900 bash -c "$(declare -f T); T 4 --mode strong --grid $g --steps 10 --warmup 5 --no-e2e" > gpurun_out/final6/strong_n4_$g.json 2> gpurun_out/final6/strong_n4_$g.err; done
timeout 900 bash -c "$(declare -f T); T 4 --steps 20 --warmup 5 --no-e2e --transport nccl" > gpurun_out/final6/weak_n4_nccl.json 2> gpurun_out/final6/weak_n4_nccl.err
timeout 900 bash -c "$(declare -f T); T 4 --mode strong --steps 10 --warmup 5 --no-e2e --depth 2" > gpurun_out/final6/strong_n4_depth2.json 2> gpurun_out/final6/strong_n4_depth2.err
timeout 300 python tools/sim_bench.py --gpus 4 --grid 4x1x1 --steps 20 > gpurun_out/final6/sim_weak_4x1x1.json 2>&1
timeout 300 python tools/sim_bench.py --gpus 4 --grid 2x2x1 --steps 20 > gpurun_out/final6/sim_weak_2x2x1.json 2>&1
timeout 900 python tools/adapter_e2e.py --kind heat --rank 3 --extent 1024 --order 4 --T 100 --calls 2 > gpurun_out/final6/adapter_e2e.json 2> gpurun_out/final6/adapter_e2e.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final6/reference_n1.json 2> gpurun_out/final6/reference_n1.err
echo done
