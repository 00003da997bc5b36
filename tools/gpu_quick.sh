# quick check: precise-grid parity subset + sim tests + C4 timing
mkdir -p gpurun_out
rm -f gpurun_out/parity_r02.jsonl
SMPM_PARITY_REPORT=gpurun_out/parity_r02.jsonl timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_sim.py "tests/test_gpu_configs.py::test_benchmarked_config_matches_oracle[C2-650-precise_grid]" "tests/test_gpu_configs.py::test_benchmarked_config_matches_oracle[C4-600-precise_grid]" "tests/test_gpu_configs.py::test_benchmarked_config_matches_oracle[C1-300-precise_grid]" > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_quick.log
bash tools/gpu_ab_short.sh 10 libsmpm.so
