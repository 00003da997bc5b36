mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke.log
timeout 600 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_run.py wide fast 2 > gpurun_out/race_f32.log 2>&1; echo race=$?; grep -h "RACECHECK SUMMARY\|ERROR SUMMARY" gpurun_out/race_f32.log | head
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-cold --late-steps 0 > gpurun_out/bench_f32.log 2>&1; echo bench=$?; tail -c 1500 gpurun_out/bench_f32.log
SMPM_ARENA=fixed timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-cold --late-steps 0 > gpurun_out/bench_fixed.log 2>&1; echo benchfixed=$?; tail -c 600 gpurun_out/bench_fixed.log
SMPM_PARITY_REPORT=gpurun_out/parity_r02.jsonl timeout 900 python -m pytest -q -s -m gpu tests/test_gpu_configs.py tests/test_gpu_sim.py > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
