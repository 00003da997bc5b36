# ncu --set full of k_g2p2g_ws in the late (flowing) regime of C4
mkdir -p gpurun_out
LATE=${LATE:-600}
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:g2p2g_ws -s $((LATE - 2)) -c 1 -o gpurun_out/ws_late -f python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps $LATE > gpurun_out/ncu_late_ws.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_late_ws.log
