O=gpurun_out/r1d; mkdir -p $O
for rep in 1 2 3; do HG_ONLY=pw_advection_128x512x512 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON; done > $O/pw_new.log 2>&1
timeout 600 python bench.py --workload pw_advection > $O/bench_pw_new.log 2>&1; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fuzz.py -x -q -m gpu -k "authored or pw_advection or shallow or fuzz or multi_apply" > $O/t_pw_new.log 2>&1; echo "t rc=$?"
cat $O/pw_new.log; tail -1 $O/bench_pw_new.log | cut -c1-200; tail -1 $O/t_pw_new.log
