# round-2 evidence: full GPU suite, default bench + reference arm, launch list,
# one ncu --set full of the fused kernel, all configs (incl. Simulation.run)
mkdir -p gpurun_out
S=$SECONDS; timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02d_pytest_gpu.log 2>&1; echo pytest=$? $((SECONDS-S))s; tail -3 gpurun_out/r02d_pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r02d_smoke.log
S=$SECONDS; timeout 1200 python bench.py > gpurun_out/r02d_bench.log 2> gpurun_out/r02d_bench.err; echo bench=$? $((SECONDS-S))s
S=$SECONDS; timeout 1200 python bench.py --impl reference > gpurun_out/r02d_bench_ref.log 2> gpurun_out/r02d_bench_ref.err; echo ref=$? $((SECONDS-S))s
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02d_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/r02d_launch_run.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:g2p2g_ws -s 5 -c 1 -o gpurun_out/r02d_fused python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/r02d_ncu.log 2>&1; echo ncu=$?
for c in C1 C2 C3; do timeout 600 python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/r02d_cfg_$c.log 2>&1; echo cfg $c=$?; done
