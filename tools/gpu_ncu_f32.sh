# one ncu --set full capture of the fused fast-mode kernel on C4 (steady state)
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:g2p2g -s 5 -c 1 -o gpurun_out/f32_full python bench.py --steps 2 --warmup 4 --no-cpu --no-cold --no-alt --late-steps 0 > gpurun_out/ncu_f32.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_f32.log
