# tile-geometry sweep of the heat SDO4 star (variants built with make variant ...)
for rep in 1 2; do
for v in base x32y8 x32y8m2 x32y12 x24y16 x32y16 x16y24; do
  if [ $v = base ]; then L=""; else L=paper_2404_02218_b200/lib/variants/libhalogen_b200_$v.so; fi
  echo "=== variant $v rep $rep"
  HG_LIB=$L HG_ONLY=heat3d_so4_1024,heat3d_so4_512 HG_CHUNKS=0,8,16 timeout 600 python tools/sweep.py 2>&1 | grep -v JSON
done
done
