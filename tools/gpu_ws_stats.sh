SMPM_LIB=libsmpm_stats.so timeout 600 python bench.py --no-cpu --no-cold --no-alt --late-steps 600 --steps 3 --warmup 3 > gpurun_out/wsstats.log 2>&1; echo rc=$?
grep "WSSTATS\|WSCLK" gpurun_out/wsstats.log | head -4 > gpurun_out/wsstats_first.txt; grep "WSSTATS\|WSCLK" gpurun_out/wsstats.log | tail -4 > gpurun_out/wsstats_last.txt; wc -l gpurun_out/wsstats.log
