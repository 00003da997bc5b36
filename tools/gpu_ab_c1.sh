# A/B of library builds on C1 (run() timing) and C4: bash tools/gpu_ab_c1.sh lib...
mkdir -p gpurun_out
for v in "$@"; do
  for c in C1 C4; do
    SMPM_LIB=$v timeout 600 python bench.py --config $c --no-cpu --no-cold --no-alt --late-steps 0 --steps $([ $c = C1 ] && echo 100 || echo 10) > gpurun_out/abc_${v}_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abc_${v}_$c.log').read().strip().splitlines()[-1]); print('$v $c step', round(d['ms_per_step'],4), 'run', round(d['run']['ms_per_step'],4), {k: round(x,4) for k,x in d['phases_ms'].items()})" || tail -3 gpurun_out/abc_${v}_$c.log
  done
done
