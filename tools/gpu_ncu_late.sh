# ncu --set full of the fused fast-mode kernel in the late (flowing) regime of C4:
# skip the early bench launches and the first LATE steps of the late leg
mkdir -p gpurun_out
LATE=${LATE:-600}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:g2p2g -s $((LATE - 2)) -c 1 -o gpurun_out/f32_late python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps $LATE > gpurun_out/ncu_late.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_late.log
