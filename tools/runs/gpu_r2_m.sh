# sustained (bench value) A/B: 10-slot (shipped) vs 8-slot ring on the 128x12 tile, same box
mkdir -p gpurun_out/r2_m
for rep in 1 2 3; do
  timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_m/ship_$rep.json 2>/dev/null
  HG_LIB=$PWD/paper_2404_02218_b200/lib/variants/libhalogen_b200_ring8.so timeout 600 python bench.py --steps 40 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/r2_m/ring8_$rep.json 2>/dev/null
done
echo done
