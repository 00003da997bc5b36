# one ncu --set full capture of the warp-specialised fused kernel (steady state, C4)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:g2p2g_ws -s 5 -c 1 -o gpurun_out/ws_fused -f python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/ws_ncu.log 2>&1; echo ncu=$?
