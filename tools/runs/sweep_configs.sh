# overlapped gather: bench.py per config over the number of gather SMs
for c in ${CFGS:-c1 c3 c4 c5}; do
for g in ${SMS:-0 8 16 24 32 48}; do
  ROCP_GATHER_SMS=$g timeout 300 python bench.py --no-cpu --no-e2e --config $c 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c G=$g', round(d['value']), round(d['ms_per_step'],3), 'gather', round(d['roofline']['avg_launch_ms'],3), 'chain', round(d['roofline_chain']['avg_launch_ms'],3))"
done
done
