# overlapped gather on a few SMs for the small-gather configs (model picks 0 there)
for c in c1 c3 c5; do for g in 0 4 8; do
  ROCP_GATHER_SMS=$g timeout 300 python bench.py --no-cpu --no-e2e --config $c | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$c G=$g', round(d['value']), round(d['ms_per_step'],3), 'gather', round(r['avg_launch_ms'],3), 'chain', round(d['roofline_chain']['avg_launch_ms'],3))"
done; done
