# A/B of WS-kernel build variants on C4 (early + late), then the sim tests and
# the benchmarked-config parity subset with the kernel pinned to ws
# usage: bash tools/gpu_ab_ws.sh lib...   (LATE=N late point, TESTS=0 skips tests)
mkdir -p gpurun_out
SMPM_FUSED=ws timeout 300 python -m pytest -q -x -m gpu tests/test_gpu_sim.py > gpurun_out/ws_sim.log 2>&1; echo ws_sim=$?; tail -2 gpurun_out/ws_sim.log
for v in "$@"; do
  SMPM_LIB=$v timeout 600 python bench.py --no-cpu --no-cold --no-alt --late-steps ${LATE:-600} --steps 10 > gpurun_out/ab_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); l=d.get('late') or {}; print('$v', round(d['ms_per_step'],3), 'fused', round(d['phases_ms']['fused'],3), 'late fused', round(l.get('phases_ms',{}).get('fused',0),3))" || tail -5 gpurun_out/ab_$v.log
done
if [ "${TESTS:-1}" = 1 ]; then
SMPM_FUSED=ws SMPM_PARITY_REPORT=gpurun_out/parity_ws.jsonl timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_module.py tests/test_gpu_configs.py tests/test_gpu_run.py tests/test_gpu_slabs.py > gpurun_out/pytest_ws.log 2>&1; echo pytest_ws=$?; tail -2 gpurun_out/pytest_ws.log
fi
