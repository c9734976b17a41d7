timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -2
for G in 0 1; do
if [ $G = 1 ]; then export HG_NO_GRAPH=1; fi
echo "no_graph=$G"; HG_ONLY=heat2d_so2_1024,heat3d_so4_512,pw_advection_128x512x512,heat3d_so4_1024 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
