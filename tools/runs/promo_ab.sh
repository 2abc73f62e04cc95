# TMA L2 promotion A/B for the window gather (in-step at the model's SM count, and standalone)
for p in 0 1 2; do
  ROCP_GATHER_PROMO=$p timeout 300 python bench.py --no-cpu --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('promo=$p', round(d['value']), round(d['ms_per_step'],3), 'gather', round(r['avg_launch_ms'],3), 'chain', round(d['roofline_chain']['avg_launch_ms'],3), 'standalone', round(r['standalone']['avg_launch_ms'],3))"
done
for p in 0 1; do
ROCP_GATHER_PROMO=$p ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_gather_warps -s 3 -c 2 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 | grep -E "dram__|gpu__time"
done
