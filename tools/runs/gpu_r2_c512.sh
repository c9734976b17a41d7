# config 2 (heat SDO4 512^3): z-chunk count vs wave quantisation (8 = auto: 4.65 waves of 296
# CTAs; 12: 6.97 waves), sustained bench value, alternating
mkdir -p gpurun_out/c512
for rep in 1 2; do
  for c in 8 12 10 16; do
    timeout 300 python bench.py --workload heat3d_512 --chunks $c --no-cpu-baseline --no-e2e > gpurun_out/c512/c${c}_$rep.json 2>/dev/null
  done
done
