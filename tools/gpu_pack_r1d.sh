mkdir -p gpurun_out/r1d
for rep in 1 2; do
for v in pack1 pack0; do
  if [ $v = pack1 ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v rep $rep"
  HG_LIB=$L HG_ONLY=heat3d_so4_1024,heat3d_so4_512,wave3d_so8_1024,heat2d_so2_16384 HG_CHUNKS=0 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
  HG_LIB=$L python bench.py --steps 200 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(\"bench heat3d\", round(d[\"value\"],1), d[\"clocks\"])"
done
done > gpurun_out/r1d/pack.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "serial or medium or wide or config" > gpurun_out/r1d/t_pack.log 2>&1; echo "t rc=$?"
cat gpurun_out/r1d/pack.log; tail -2 gpurun_out/r1d/t_pack.log
