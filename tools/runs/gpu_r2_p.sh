# vectorized packed put + hg_plan_bind: tests and NVLink counters of the x-face put
mkdir -p gpurun_out/r2_p gpurun_out/nvl2
timeout 1500 python -m pytest tests/test_multigpu.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "x_faces or caller_bound or deep or one_rank_per_device or simulate or two_ranks" > gpurun_out/r2_p/tests.log 2>&1
echo rc=$? >> gpurun_out/r2_p/tests.log
M="nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --devices 0 -k regex:putKernel -c 1 --metrics $M --csv python tools/nvlink_probe.py --grid 1x1x2 > gpurun_out/nvl2/put_1x1x2.csv 2> gpurun_out/nvl2/put_1x1x2.err
echo done
