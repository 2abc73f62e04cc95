# C4: device throughput against the gather's SM count (the gather paces the wide chain)
for g in ${C4_SWEEP:-0 29 40 52 64 74}; do
  ROCP_GATHER_SMS=$g timeout 600 python bench.py --config c4 --no-cpu --no-e2e --steps 5 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']; c=d.get('roofline_chain') or {}
print('G', $g, 'value', round(d['value']), 'ms', round(d['ms_per_step'],3), 'gather_ms', r.get('avg_launch_ms'), 'sms', r.get('sms'), 'chain_ms', c.get('avg_launch_ms'))"
done
