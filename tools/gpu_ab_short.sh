# quick A/B of build variants (bench only, few steps): bash tools/gpu_ab_short.sh STEPS lib...
mkdir -p gpurun_out
st=$1; shift
for v in "$@"; do
  timeout 600 env SMPM_LIB=$v python bench.py --no-cpu --no-cold --no-alt --late-steps ${LATE:-0} --steps $st > gpurun_out/ab_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/ab_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), {k: round(x,3) for k,x in d['phases_ms'].items()})" || tail -5 gpurun_out/ab_$v.log
done
