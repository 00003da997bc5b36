# C1 (granular column, 128k particles): per-kernel durations of batched steps
# (ncu launch list) next to the run() timing, to split kernel time from gaps
mkdir -p gpurun_out
timeout 600 python bench.py --config C1 --steps 50 --warmup 5 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/c1_bench.log 2>&1; echo bench=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c1_launches.csv python bench.py --config C1 --steps 20 --warmup 3 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/c1_launch_run.log 2>&1; echo launches=$?
