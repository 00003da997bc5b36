# Round evidence (run under gpurun): smoke, GPU tests, bench (ours + reference arm),
# ncu launch list of the bench, ncu --set full of one steady-state fused launch.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/b_ncu.log 2>&1; echo ncu1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:g2p2g -s 5 -c 1 -o gpurun_out/fused_full python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/b_ncu2.log 2>&1; echo ncu2=$?
for f in smoke pytest_gpu bench bench_ref; do echo "== $f"; tail -n 3 gpurun_out/$f.log; done
# late-time regime (10 % of C4, 600 steps): timing and one ncu capture of the fused kernel
timeout 900 python tools/late_profile.py 600 > gpurun_out/late.log 2>&1; echo late=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:g2p2g -s 590 -c 1 -o gpurun_out/late590 python tools/late_profile.py 600 > gpurun_out/late590.log 2>&1; echo ncu3=$?
tail -n 4 gpurun_out/late.log
