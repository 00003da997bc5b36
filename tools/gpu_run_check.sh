mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_run.py tests/test_gpu_sim.py > gpurun_out/pytest_run.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_run.log
for c in C1 C2 C3; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/cfg_$c.log 2>&1; python -c "import json; d=json.loads(open('gpurun_out/cfg_$c.log').read().strip().splitlines()[-1]); print('$c', d['config']['n_particles'], 'step ms', round(d['ms_per_step'],4), 'run ms', round(d['run']['ms_per_step'],4), d['phases_ms'])" || tail -5 gpurun_out/cfg_$c.log; done
bash tools/gpu_ab_short.sh 10 libsmpm.so
