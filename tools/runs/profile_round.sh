# bench line + ncu launch list + ncu --set full of the window gather (in-step) and of the
# dataflow chain (k_flow), configs[1]
set -e
python bench.py > gpurun_out/bench_full.log 2>&1; tail -1 gpurun_out/bench_full.log | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_gather_warps -s 3 -c 2 -o gpurun_out/gather_warps \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/ncu_gather.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_flow -s 3 -c 1 -o gpurun_out/flow \
    python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/ncu_flow.log 2>&1
ls -la gpurun_out
