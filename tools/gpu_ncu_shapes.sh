for S in 1024,1024,1024 1024,1024,64 1024,16,1024 16384,16,64 4096,512,512; do
python tools/prof_shape.py --shape $S > /dev/null 2>&1 && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --clock-control none -k regex:starKernel -s 2 -c 1 python tools/prof_shape.py --shape $S 2>&1 | grep -E "dram__|gpu__time|lts__" | sed "s/^/$S /"
done
