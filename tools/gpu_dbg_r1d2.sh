mkdir -p gpurun_out/r1d
L=gpurun_out/r1d/dbg2.log; : > $L
T=1 timeout 300 python tools/debug_flux_unfused.py >> $L 2>&1
HG_JIT_DEPTH=1 timeout 300 python tools/debug_flux_unfused.py >> $L 2>&1
HG_JIT_DEPTH=20 timeout 300 python tools/debug_flux_unfused.py >> $L 2>&1
HG_MULTI_NODIRECT=1 timeout 300 python tools/debug_flux_unfused.py >> $L 2>&1
for tool in racecheck synccheck memcheck initcheck; do
  REPS=2 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/debug_flux_unfused.py > gpurun_out/r1d/san_$tool.log 2>&1; echo "$tool rc=$?" >> $L
done
cat $L; tail -30 gpurun_out/r1d/san_*.log
