# compute-sanitizer evidence: memcheck / racecheck / synccheck over the
# star kernels (heat SDO4, wave SDO8, 2D), the resident 2D kernel, the generated fused-apply
# kernel, the put / flag kernels, and the fused NVLink put on 2 ranks (small shapes: the tools
# instrument every access)
mkdir -p gpurun_out/sanitizer
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 50 --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer/smoke_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/smoke_$tool.log
done
timeout 1200 $CS --tool memcheck --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/cases_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/cases_memcheck.log
timeout 1200 $CS --tool racecheck --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/cases_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/cases_racecheck.log
timeout 1200 $CS --tool synccheck --print-limit 50 --error-exitcode 9 python tools/sanitize_cases.py > gpurun_out/sanitizer/cases_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/sanitizer/cases_synccheck.log
# two ranks over NVLink: the fused put, flags, packed x slabs, handshake (memcheck per rank)
for grid in 2x1x1 1x1x2; do
  timeout 1200 python -m torch.distributed.run --standalone --nproc-per-node 2 --no-python $CS --tool memcheck --print-limit 50 --error-exitcode 9 python tools/dmp_check.py --kind heat --rank 3 --extents 96x40x64 --order 4 --grid $grid --T 4 --calls 1,3 --upload > gpurun_out/sanitizer/dmp_${grid}_memcheck.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitizer/dmp_${grid}_memcheck.log
done
echo done
