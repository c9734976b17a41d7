mkdir -p gpurun_out/r1d
timeout 600 python tools/debug_flux_unfused.py > gpurun_out/r1d/dbg_flux.log 2>&1; echo "dbg rc=$?"
timeout 300 python tools/xfer_probe.py > gpurun_out/r1d/xfer.log 2>&1; echo "xfer rc=$?"
cat gpurun_out/r1d/dbg_flux.log gpurun_out/r1d/xfer.log
