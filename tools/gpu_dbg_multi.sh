O=gpurun_out/r1m; mkdir -p $O; : > $O/dbg_multi.log
A="--kind heat --rank 3 --extent 100 --order 8 --T 6 --calls 4,2"
for v in hint nohint; do
  if [ $v = hint ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  for cfg in "2 none" "4 2x2x1" "4 1x2x2" "4 4x1x1"; do
    set -- $cfg; G=""; [ $2 != none ] && G="--grid $2"
    echo "=== $v nproc=$1 grid=$2" >> $O/dbg_multi.log
    HG_LIB=$L timeout 300 python -m torch.distributed.run --standalone --nproc-per-node $1 tools/dmp_check.py $A $G > $O/dbg_out.txt 2>&1; echo "rc=$?" >> $O/dbg_multi.log
    grep -E "OK|rror|CUDA|mismatch|differ" $O/dbg_out.txt | grep -v "TORCH_USE_CUDA_DSA\|CUDA_LAUNCH_BLOCKING" | head -8 >> $O/dbg_multi.log
  done
done
cat $O/dbg_multi.log
