O=gpurun_out/r1d; mkdir -p $O
for cfg in "1 6" "2 2" "2 3" "3 1" "3 2" "2 1"; do
set -- $cfg
echo "minb=$1 depth=$2"; HG_JIT_MINB=$1 HG_JIT_DEPTH=$2 HG_ONLY=pw_advection_128x512x512 HG_CHUNKS=0,1,8 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON
done > $O/pw_sweep2.log 2>&1
cat $O/pw_sweep2.log
