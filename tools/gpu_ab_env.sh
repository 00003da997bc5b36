# A/B of an environment switch on C4 (early + late): bash tools/gpu_ab_env.sh "VAR=a" "VAR=b" ...
mkdir -p gpurun_out
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 600 python bench.py --no-cpu --no-cold --no-alt --late-steps ${LATE:-600} --steps 10 > gpurun_out/abenv_$i.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/abenv_$i.log').read().strip().splitlines()[-1]); l=d.get('late') or {}; print('$e', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, 'late', round(l.get('ms_per_step',0),3))" || tail -5 gpurun_out/abenv_$i.log
done
