# iteration check: C4 A/B timing of build variants + the precise-grid parity subset
# usage: bash tools/gpu_iter.sh [lib ...]   (TESTS=0 skips the tests, LATE=N adds a late-time point)
mkdir -p gpurun_out
libs="${@:-libsmpm.so}"
bash tools/gpu_ab_short.sh 10 $libs
if [ "${TESTS:-1}" = 1 ]; then
rm -f gpurun_out/parity_iter.jsonl
SMPM_PARITY_REPORT=gpurun_out/parity_iter.jsonl timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_sim.py tests/test_gpu_configs.py > gpurun_out/pytest_iter.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_iter.log
fi
