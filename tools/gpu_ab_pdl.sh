# PDL A/B: C1 and C4 run() timing with SMPM_PDL=1/0, then the batched-step and sim tests
mkdir -p gpurun_out
for e in SMPM_PDL=1 SMPM_PDL=0 SMPM_PDL=1 SMPM_PDL=0; do
  for c in C1 C4; do
    env $e timeout 600 python bench.py --config $c --no-cpu --no-cold --no-alt --late-steps 0 --steps $([ $c = C1 ] && echo 100 || echo 10) > gpurun_out/pdl_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/pdl_$c.log').read().strip().splitlines()[-1]); print('$e $c step', round(d['ms_per_step'],4), 'run', round(d['run']['ms_per_step'],4))" || tail -3 gpurun_out/pdl_$c.log
  done
done
timeout 1500 python -m pytest -q -x -m gpu tests/test_gpu_run.py tests/test_gpu_sim.py tests/test_gpu_ws.py > gpurun_out/pt_pdl.log 2>&1; echo pt=$?; tail -2 gpurun_out/pt_pdl.log
