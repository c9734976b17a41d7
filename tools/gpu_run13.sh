for W in heat3d_weak heat3d_512 wave3d_1024 pw_advection heat2d_1024; do
timeout 600 python bench.py --workload $W > gpurun_out/bench_$W.log 2>&1; echo "$W rc=$?"; tail -1 gpurun_out/bench_$W.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('  value %.1f %s ms/step %.4f frac %.3f clocks %s e2e %.1f cpu %s' % (d['value'], d['unit'], d['ms_per_step'], r['frac'], d['clocks'], d['e2e']['value'] if d.get('e2e') else -1, d.get('cpu_baseline',{}).get('value')))"
done
