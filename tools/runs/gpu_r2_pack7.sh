# config 5 sustained (bench value, 400 timed steps) by z-chunk count: 8 / 12 / 16 (auto) / 24
mkdir -p gpurun_out/pack7
for rep in 1 2; do
  for c in 16 8 12 24; do
    timeout 600 python bench.py --chunks $c --no-cpu-baseline --no-e2e > gpurun_out/pack7/c${c}_$rep.json 2>/dev/null
  done
done
