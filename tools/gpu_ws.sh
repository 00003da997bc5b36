# warp-specialised fused kernel: smoke under a short timeout, A/B timing on C4
# (SMPM_FUSED=cta|ws), then the parity subset with the kernel pinned to ws
mkdir -p gpurun_out
SMPM_FUSED=ws timeout 300 python -m pytest -q -x -m gpu tests/test_gpu_sim.py > gpurun_out/ws_sim.log 2>&1; echo ws_sim=$?; tail -3 gpurun_out/ws_sim.log
for v in ${VARIANTS:-cta ws}; do
  SMPM_FUSED=$v timeout 600 python bench.py --no-cpu --no-cold --no-alt --late-steps ${LATE:-0} --steps 10 > gpurun_out/ab_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phases_ms'].items()}, d.get('late',{}).get('phases_ms'))" || tail -5 gpurun_out/ab_$v.log
done
if [ "${TESTS:-1}" = 1 ]; then
SMPM_FUSED=ws SMPM_PARITY_REPORT=gpurun_out/parity_ws.jsonl timeout 1200 python -m pytest -q -x -m gpu tests/test_gpu_configs.py tests/test_gpu_run.py > gpurun_out/pytest_ws.log 2>&1; echo pytest_ws=$?; tail -3 gpurun_out/pytest_ws.log
fi
