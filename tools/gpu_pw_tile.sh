O=gpurun_out/r1d; mkdir -p $O
for cfg in "16 16 6" "16 16 3" "16 24 3" "16 32 2" "16 32 3" "32 8 3" "32 8 6" "32 16 2" "32 16 3" "32 12 3"; do
set -- $cfg
echo -n "txt=$1 tyt=$2 depth=$3 "; HG_JIT_TXT=$1 HG_JIT_TYT=$2 HG_JIT_DEPTH=$3 HG_ONLY=pw_advection_128x512x512 HG_CHUNKS=0,8 timeout 300 python tools/sweep.py 2>&1 | grep -v JSON | tr '\n' ' '; echo
done > $O/pw_tile.log 2>&1
HG_JIT_TXT=32 HG_JIT_TYT=8 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "authored or pw_advection or shallow" > $O/t_pw_tile.log 2>&1; echo "t rc=$?"
cat $O/pw_tile.log; tail -1 $O/t_pw_tile.log
