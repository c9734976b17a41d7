# resident 2D: steps per exchange K (1/2/3/4) with the register-sourced exchange, same box
mkdir -p gpurun_out/r2_q
V=$PWD/paper_2404_02218_b200/lib/variants
for rep in 1 2; do
  timeout 300 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_q/k2_$rep.json 2>/dev/null
  for k in 1 3 4; do HG_LIB=$V/libhalogen_b200_resk$k.so timeout 300 python bench.py --workload heat2d_1024 --steps 400 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_q/k${k}_$rep.json 2>/dev/null; done
done
echo done
