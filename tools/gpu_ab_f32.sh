# A/B of the fused fast-mode kernel: fp32 arena vs int32 fixed point (C4), plus
# one ncu --set full capture of the fp32 kernel and the sim GPU tests
mkdir -p gpurun_out
for arena in f32 fixed; do
  if [ $arena = fixed ]; then export SMPM_ARENA=fixed; else unset SMPM_ARENA; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-cold --no-alt --late-steps ${LATE:-0} > gpurun_out/ab_$arena.log 2>&1
  python - gpurun_out/ab_$arena.log $arena <<'PY'
import json, sys
l = [x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[2], "FAILED", open(sys.argv[1]).read()[-800:]); sys.exit()
d = json.loads(l[-1])
late = d.get("late") or {}
print(sys.argv[2], "ms/step %.3f" % d["ms_per_step"], "phases", {k: round(v, 3) for k, v in d["phases_ms"].items()},
      "frac %.3f" % d["roofline"]["frac"], "late", {k: late.get(k) for k in ("ms_per_step", "phases_ms")} if late else None)
PY
done
unset SMPM_ARENA
if [ "${NCU:-1}" = 1 ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:g2p2g -s 5 -c 1 -o gpurun_out/f32_full python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/ncu_f32.log 2>&1; echo ncu=$?
fi
if [ "${TESTS:-0}" = 1 ]; then
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_sim.py tests/test_gpu_configs.py > gpurun_out/pytest_ab.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab.log
fi
