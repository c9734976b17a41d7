for c in 1 3 8 24; do
python tools/prof_star.py --chunks $c > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py --chunks $c 2>&1 | grep -E "dram__|gpu__time|lts__|sm__cycles" | sed "s/^/chunks=$c /"
done
python tools/prof_star.py --kind wave --order 8 > /dev/null 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_star.py --kind wave --order 8 2>&1 | grep -E "dram__|gpu__time" | sed "s/^/wave /"
