# Round-2 final evidence: bench lines (ours + reference arm), ncu launch list of the bench step,
# ncu --set full of the dataflow chain (configs[1]) and of the wide chain (configs[3]), C4 phase
# trace and gather-split sweep, fp64-MMA occupancy and inner-loop microbenchmarks.
set -x
O=gpurun_out/final
mkdir -p $O
python bench.py > $O/bench_full.log 2>&1; tail -1 $O/bench_full.log > $O/bench_line.json
python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.log 2>&1; tail -1 $O/bench_ref.log > $O/bench_reference_line.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_step.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_flow -s 3 -c 1 -o $O/flow \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_flow.log 2>&1
ncu -i $O/flow.ncu-rep --page details > $O/ncu_flow_details.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather_warps -s 3 -c 1 -o $O/gather \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > $O/ncu_gather.log 2>&1
ncu -i $O/gather.ncu-rep --page details > $O/ncu_gather_details.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_chain -s 2 -c 1 -o $O/chain_c4 \
    python bench.py --config c4 --steps 1 --warmup 2 --no-cpu --no-e2e --no-configs > $O/ncu_chain_c4.log 2>&1
ncu -i $O/chain_c4.ncu-rep --page details > $O/ncu_chain_c4_details.txt 2>&1
python tools_trace.py '{"dims":[4000,4000,500],"R":50,"t_init":50,"B":50}' > $O/trace_c4.txt 2>&1
ROCP_GATHER_SMS=0 python tools_trace.py '{"dims":[4000,4000,500],"R":50,"t_init":50,"B":50}' > $O/trace_c4_serial_gather.txt 2>&1
python tools/runs/flow_trace.py c2 > $O/flow_trace_c2.txt 2>&1
tools/dmma_occ > $O/dmma_occupancy.txt 2>&1
tools/stream_bench > $O/stream_inner_loop.txt 2>&1
python tools/runs/multi_stream.py c2 1 2:60 3:40 4:30 6:20 > $O/multi_stream_c2.txt 2>&1
rm -f $O/*.ncu-rep
ls -la $O
