# bench (ours, full default run) + reference arm
mkdir -p gpurun_out
free -g | head -2
S=$SECONDS; timeout 1200 python bench.py > gpurun_out/bench.log 2> gpurun_out/bench.err; echo bench=$? wall=$((SECONDS-S))s
tail -c 5000 gpurun_out/bench.log; tail -3 gpurun_out/bench.err
S=$SECONDS; timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err; echo ref=$? wall=$((SECONDS-S))s
tail -c 1500 gpurun_out/bench_ref.log; tail -3 gpurun_out/bench_ref.err
