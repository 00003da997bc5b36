# slab tests (new frame exchange + rebalancing), then all configs' timings
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_slabs.py > gpurun_out/pytest_slabs.log 2>&1; echo slabs=$?; tail -3 gpurun_out/pytest_slabs.log
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/cfg_$c.log 2>&1
  python - gpurun_out/cfg_$c.log $c <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], "FAILED", open(sys.argv[1]).read()[-600:]); sys.exit()
d = json.loads(l[-1])
print(sys.argv[2], d["config"]["n_particles"], "ms/step %.4f" % d["ms_per_step"], "value %.3e" % d["value"],
      {k: round(v, 4) for k, v in d["phases_ms"].items()}, "frac %.3f" % d["roofline"]["frac"])
PY
done
