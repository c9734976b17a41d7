# NVLink counters of the fused swap (one process, two GPUs, ncu on device 0 only)
mkdir -p gpurun_out/nvl
M="nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 300 python tools/nvlink_probe.py --grid 2x1x1 > gpurun_out/nvl/plain_2x1x1.log 2>&1
for g in 2x1x1 1x1x2; do
  timeout 600 ncu --devices 0 -k regex:starKernel -s 2 -c 1 --metrics $M --csv python tools/nvlink_probe.py --grid $g > gpurun_out/nvl/star_$g.csv 2> gpurun_out/nvl/star_$g.err
  timeout 600 ncu --devices 0 -k regex:putKernel -c 1 --metrics $M --csv python tools/nvlink_probe.py --grid $g > gpurun_out/nvl/put_$g.csv 2> gpurun_out/nvl/put_$g.err
done
echo done
