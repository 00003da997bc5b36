# bench.py on every BASELINE config (C1..C4) on one GPU -> gpurun_out/cfg_*.log
mkdir -p gpurun_out
for c in C1 C2 C3 C4; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/cfg_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/cfg_$c.log').read().strip().splitlines()[-1]); print('$c', d['config']['n_particles'], round(d['ms_per_step'],3), '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], 'frac %.3f'%d['roofline']['frac'], 'cpu %.3e'%d.get('cpu_baseline',{}).get('value',0))" || tail -3 gpurun_out/cfg_$c.log
done
