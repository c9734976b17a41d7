for p in 0 1 2 3; do
  echo "=== L2 promotion $p"
  HG_L2PROMO=$p HG_ONLY=heat3d_so4_1024,wave3d_so8_1024 HG_CHUNKS=3,8,16,24,32,48 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
