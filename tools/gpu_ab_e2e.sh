# A/B of library builds on the C4 bench incl. the warm e2e leg: bash tools/gpu_ab_e2e.sh lib...
mkdir -p gpurun_out
for v in "$@"; do
  SMPM_LIB=$v timeout 900 python bench.py --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/abe_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abe_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3), 'e2e %.3e' % d['e2e']['value'], d['e2e']['rank0_breakdown'])" || tail -3 gpurun_out/abe_$v.log
done
