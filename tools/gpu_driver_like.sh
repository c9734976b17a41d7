O=gpurun_out/r1x; mkdir -p $O
t0=$(date +%s); timeout 900 python bench.py --impl reference > $O/ref_default.log 2> $O/ref_default.err; echo "ref rc=$? $(( $(date +%s) - t0 )) s"
t0=$(date +%s); timeout 900 python bench.py > $O/ours_default.log 2> $O/ours_default.err; echo "ours rc=$? $(( $(date +%s) - t0 )) s"
tail -1 $O/ref_default.log | cut -c1-250; tail -1 $O/ours_default.log | cut -c1-250
