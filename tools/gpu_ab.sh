# A/B timing of build variants + full GPU test suite (run under gpurun)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
for v in "$@"; do
  timeout 600 env SMPM_LIB=$v python bench.py --no-cpu --steps 20 > gpurun_out/ab_$v.log 2>&1; echo $v=$?
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['phases_ms'], d['value'])" || tail -5 gpurun_out/ab_$v.log
done
tail -5 gpurun_out/pytest_gpu.log
