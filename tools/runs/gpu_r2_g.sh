# round 2: full GPU suite under HG_DEBUG_GUARDS (canary bands around every device buffer: the
# out-of-bounds-write check, compute-sanitizer being closed on this pool) + resident A/B
mkdir -p gpurun_out/r2_g
for v in A B base; do
  case $v in A) L="";; B) L=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_resB.so;; base) L=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_r2base.so;; esac
  HG_LIB=$L timeout 600 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_g/heat2d_$v.json 2> gpurun_out/r2_g/heat2d_$v.err
done
HG_DEBUG_GUARDS=1 timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=5 > gpurun_out/r2_g/tests_guards.log 2>&1
echo rc=$? >> gpurun_out/r2_g/tests_guards.log
echo done
