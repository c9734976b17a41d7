# tile-geometry sweep of the wave SDO8 star
for rep in 1 2; do
for v in w16y24 w32y12 w16y28 w24y20 w32y15 w16y24d7 w32y12d7; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v rep $rep"
  HG_LIB=$L HG_ONLY=wave3d_so8_1024 HG_CHUNKS=0,8 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
done
