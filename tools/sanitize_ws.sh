mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck; do
  log=gpurun_out/sanitize/${tool}_ws.log; extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  SMPM_MODE=fast SMPM_FUSED=ws SMPM_WS_BLOCKS=4 timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $log 2>&1
  echo "$tool ws rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(tail -1 $log | cut -c1-80)"
done
