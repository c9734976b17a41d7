O=gpurun_out/r1z; mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/gpu_tests_4gpu.log 2>&1; echo "tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > $O/bench_n1.log 2>&1; echo "n1 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29554 bench.py --gpus 4 > $O/bench_weak_n4.log 2>&1; echo "weak4 rc=$?"
tail -2 $O/gpu_tests_4gpu.log; cat $O/smoke.log
for f in $O/bench_*.log; do echo "$f: $(tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d.get('clocks',{}).get('sm_mhz'))" 2>&1 | tail -1)"; done
