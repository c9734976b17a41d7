# Resident 2D kernel with packed adds: parity, then config 1 bench against the scalar variant
mkdir -p gpurun_out/pack4
V=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_scalar.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "resident or heat2d or 2d" > gpurun_out/pack4/tests.log 2>&1; echo rc=$? >> gpurun_out/pack4/tests.log
for rep in 1 2 3; do
  timeout 600 python bench.py --workload heat2d_1024 --no-cpu-baseline --no-e2e > gpurun_out/pack4/pack_$rep.json 2>/dev/null
  HG_LIB=$V timeout 600 python bench.py --workload heat2d_1024 --no-cpu-baseline --no-e2e > gpurun_out/pack4/scalar_$rep.json 2>/dev/null
done
