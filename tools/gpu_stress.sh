O=gpurun_out/r1s; mkdir -p $O
for i in 1 2 3; do
timeout 900 python -m pytest tests/test_fuzz.py tests/test_gpu_parity.py -q -m gpu -k "fuzz or authored or shallow or multi_apply or serial or wide or resident" > $O/stress_$i.log 2>&1; echo "rep $i rc=$?"; tail -1 $O/stress_$i.log
done
