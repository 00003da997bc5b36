# compute-sanitizer evidence (run under gpurun): memcheck / racecheck /
# synccheck of every kernel of the step (k_scan1/2, k_bin, k_grid, the fused
# kernel in each variant, k_prologue_keys, the module kernels of the first
# prologue) on a 16k-particle moving column, 3 steps each.
#   precise : k_g2p2g_f32 (fast mode, small scenes)
#   ws      : k_g2p2g_ws (fast mode, large scenes), 4 CTAs: ~8 items per CTA
#   fixed-* : k_g2p2g int32 fixed point (precise_grid=False), narrow / wide items
#   det-*   : k_g2p2g int64 fixed point (deterministic), narrow / wide items
mkdir -p gpurun_out/sanitize
run() {  # name env... -- args
  name=$1; shift
  for tool in memcheck racecheck synccheck; do
    log=gpurun_out/sanitize/${tool}_${name}.log
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    env "$@" timeout 1200 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_run.py > $log 2>&1
    echo "$tool $name rc=$? $(grep -h 'ERROR SUMMARY\|RACECHECK SUMMARY' $log | tr '\n' ' ') $(tail -1 $log | cut -c1-80)"
  done
}
{
run precise SMPM_MODE=fast SMPM_FUSED=cta
run ws SMPM_MODE=fast SMPM_FUSED=ws SMPM_WS_BLOCKS=4
run fixed-narrow SMPM_MODE=fast SMPM_ARENA=fixed SMPM_ITEM_LAYOUT=narrow
run fixed-wide SMPM_MODE=fast SMPM_ARENA=fixed SMPM_ITEM_LAYOUT=wide
run det-narrow SMPM_MODE=det SMPM_ITEM_LAYOUT=narrow
run det-wide SMPM_MODE=det SMPM_ITEM_LAYOUT=wide
} | tee gpurun_out/sanitize/summary.txt
