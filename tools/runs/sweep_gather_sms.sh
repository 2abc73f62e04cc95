# overlapped gather: GPU tests, then bench.py over the number of gather SMs (TMA on / off)
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for t in 1 0; do
for g in ${SMS:-0 8 12 16 20 24 32}; do
  ROCP_GATHER_TMA=$t ROCP_GATHER_SMS=$g timeout 120 python bench.py --no-cpu --no-e2e ${BENCH_ARGS:-} 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tma=$t G=$g', round(d['value']), round(d['ms_per_step'],3), 'gather', round(d['roofline']['avg_launch_ms'],3), 'chain', round(d['roofline_chain']['avg_launch_ms'],3))"
done
done
