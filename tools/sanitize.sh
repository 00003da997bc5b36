# compute-sanitizer evidence (run under gpurun): racecheck / synccheck /
# memcheck of every kernel of the fused step (k_scan1/2, k_bin, k_grid,
# k_g2p2g narrow/wide x fast/deterministic, k_prologue_keys) on a 16k scene.
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  for layout in narrow wide; do
    for mode in fast det; do
      log=gpurun_out/sanitize/${tool}_${layout}_${mode}.log
      extra=""
      [ $tool = racecheck ] && extra="--racecheck-report all"
      timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py $layout $mode 3 > $log 2>&1
      echo "$tool $layout $mode rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ')"
    done
  done
done | tee gpurun_out/sanitize/summary.txt
