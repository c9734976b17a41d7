mkdir -p gpurun_out/r2_t
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "resident or config1 or caller_bound or zero_steps" > gpurun_out/r2_t/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_t/tests.log
for rep in 1 2 3; do
  timeout 300 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_t/new_$rep.json 2>/dev/null
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_resprev.so timeout 300 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_t/prev_$rep.json 2>/dev/null
done
echo done
