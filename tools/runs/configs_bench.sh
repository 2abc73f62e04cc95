# bench.py on all five BASELINE configs (device stream + e2e) and the sharded stream at world 1
for c in c1 c2 c3 c5; do
  timeout 600 python bench.py --config $c --no-cpu > gpurun_out/cfg_$c.log 2>&1
done
timeout 900 python bench.py --config c4 --no-cpu --e2e-steps 1 > gpurun_out/cfg_c4.log 2>&1
for c in c2 c4 c5; do
  timeout 600 python bench.py --config $c --sharded --no-cpu --no-e2e > gpurun_out/cfg_${c}_sharded.log 2>&1
done
for f in gpurun_out/cfg_*.log; do
  tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; e=d.get('e2e') or {}; print('$f'.split('/')[-1], d['config']['workload'][:40], 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'e2e', round(e['value']) if e else None, 'G', r.get('sms'), 'gather_ms', round(r['avg_launch_ms'],3) if r.get('avg_launch_ms') else None, 'chain_ms', round(d['roofline_chain']['avg_launch_ms'],3) if d.get('roofline_chain') else None)"
done
