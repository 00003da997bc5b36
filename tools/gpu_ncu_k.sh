# ncu --set full of one steady-state launch of kernel regex $2 (C4) -> gpurun_out/$1.ncu-rep
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s ${3:-5} -c 1 -o gpurun_out/$1 python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/$1.log 2>&1; echo ncu=$?
