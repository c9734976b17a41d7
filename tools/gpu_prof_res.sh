mkdir -p gpurun_out/r1d
python tools/prof_resident.py > gpurun_out/r1d/plain_res.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:residentKernel -s 2 -c 1 -o gpurun_out/r1d/prof_resident python tools/prof_resident.py > gpurun_out/r1d/ncu_res.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r1d/ncu_res.log
