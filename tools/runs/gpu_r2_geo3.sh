# two output rows per thread (GEO 3, 128x16 tile): parity (forced), then same-box A/B against
# the shipped 128x12 tile (GEO 1) -- burst (sweep.py) and sustained (bench.py) at 1024^3, 512^3
mkdir -p gpurun_out/geo3
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "two_row or wide_tile" > gpurun_out/geo3/tests.log 2>&1; echo rc=$? >> gpurun_out/geo3/tests.log
grep -q "rc=0" gpurun_out/geo3/tests.log || exit 0
export HG_ONLY=heat3d_so4_1024,heat3d_so4_512
for rep in 1 2; do
  for g in 1 3; do HG_STAR_GEO=$g python tools/sweep.py > gpurun_out/geo3/sweep_g${g}_$rep.log 2>&1; done
done
for rep in 1 2; do
  for g in 1 3; do
    HG_STAR_GEO=$g timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/geo3/bench_g${g}_$rep.json 2>/dev/null
    HG_STAR_GEO=$g timeout 600 python bench.py --workload heat3d_512 --no-cpu-baseline --no-e2e > gpurun_out/geo3/bench512_g${g}_$rep.json 2>/dev/null
  done
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,lts__t_bytes.sum
for g in 1 3; do HG_STAR_GEO=$g ncu --metrics $M --clock-control none -k regex:starKernel -s 2 -c 3 --csv python tools/prof_star.py --steps 6 > gpurun_out/geo3/ncu_g$g.csv 2>&1; done
